// cc_armc_s6.cu — constant slot 6 of the constant-bank ARM (cc_armc.cuh).
#define CCB_ARMC_SLOT 6
#include "cc_armc.cuh"
