// cc_armc_s3.cu — constant slot 3 of the constant-bank ARM (cc_armc.cuh).
#define CCB_ARMC_SLOT 3
#include "cc_armc.cuh"
