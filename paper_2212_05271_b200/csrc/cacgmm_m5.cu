// cACGMM EM / MVDR-statistics kernels for M = 5 channels.
#define GSS_M 5
#include "cacgmm_inst.inc"
