// cACGMM EM / MVDR-statistics kernels for M = 4 channels.
#define GSS_M 4
#include "cacgmm_inst.inc"
