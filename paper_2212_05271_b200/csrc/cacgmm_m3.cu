// cACGMM EM / MVDR-statistics kernels for M = 3 channels.
#define GSS_M 3
#include "cacgmm_inst.inc"
