// cc_armc_s7.cu — constant slot 7 of the constant-bank ARM (cc_armc.cuh).
#define CCB_ARMC_SLOT 7
#include "cc_armc.cuh"
