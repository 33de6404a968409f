// cACGMM EM / MVDR-statistics kernels for M = 8 channels.
#define GSS_M 8
#include "cacgmm_inst.inc"
