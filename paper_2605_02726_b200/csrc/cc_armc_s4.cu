// cc_armc_s4.cu — constant slot 4 of the constant-bank ARM (cc_armc.cuh).
#define CCB_ARMC_SLOT 4
#include "cc_armc.cuh"
