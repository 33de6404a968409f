// cACGMM EM / MVDR-statistics kernels for M = 2 channels.
#define GSS_M 2
#include "cacgmm_inst.inc"
