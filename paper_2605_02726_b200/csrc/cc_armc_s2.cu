// cc_armc_s2.cu — constant slot 2 of the constant-bank ARM (cc_armc.cuh).
#define CCB_ARMC_SLOT 2
#include "cc_armc.cuh"
