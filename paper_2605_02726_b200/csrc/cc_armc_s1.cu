// cc_armc_s1.cu — constant slot 1 of the constant-bank ARM (cc_armc.cuh).
#define CCB_ARMC_SLOT 1
#include "cc_armc.cuh"
