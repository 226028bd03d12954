// cc_armc_s5.cu — constant slot 5 of the constant-bank ARM (cc_armc.cuh).
#define CCB_ARMC_SLOT 5
#include "cc_armc.cuh"
