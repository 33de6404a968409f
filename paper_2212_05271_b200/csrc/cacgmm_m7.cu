// cACGMM EM / MVDR-statistics kernels for M = 7 channels.
#define GSS_M 7
#include "cacgmm_inst.inc"
