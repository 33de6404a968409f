// cACGMM EM / MVDR-statistics kernels for M = 6 channels.
#define GSS_M 6
#include "cacgmm_inst.inc"
