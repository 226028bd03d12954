// cc_armc_s0.cu — constant slot 0 of the constant-bank ARM (cc_armc.cuh).
#define CCB_ARMC_SLOT 0
#include "cc_armc.cuh"
