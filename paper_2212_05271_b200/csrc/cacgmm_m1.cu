// cACGMM EM / MVDR-statistics kernels for M = 1 channels.
#define GSS_M 1
#include "cacgmm_inst.inc"
