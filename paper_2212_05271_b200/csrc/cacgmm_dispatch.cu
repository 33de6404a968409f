// cacgmm_dispatch.cu -- routes (M, KT) to the per-channel-count translation units.
#include "kernels.h"

namespace gssb {

#define GSS_DECL(m)                                                                                         \
  cudaError_t launch_em_pass_m##m(int, bool, const EmPassArgs&, int, int, cudaStream_t);                   \
  cudaError_t launch_em_update_m##m(int, const EmUpdateArgs&, int, cudaStream_t);                          \
  cudaError_t launch_mvdr_stats_m##m(int, const StatsPassArgs&, int, int, cudaStream_t);                   \
  cudaError_t launch_mvdr_stats_final_m##m(int, const StatsFinalArgs&, int, cudaStream_t);
GSS_DECL(1) GSS_DECL(2) GSS_DECL(3) GSS_DECL(4) GSS_DECL(5) GSS_DECL(6) GSS_DECL(7) GSS_DECL(8)

#define GSS_M_SWITCH(FN, ...)                     \
  switch (s.M) {                                  \
    case 1: return FN##1(s.KT, __VA_ARGS__);      \
    case 2: return FN##2(s.KT, __VA_ARGS__);      \
    case 3: return FN##3(s.KT, __VA_ARGS__);      \
    case 4: return FN##4(s.KT, __VA_ARGS__);      \
    case 5: return FN##5(s.KT, __VA_ARGS__);      \
    case 6: return FN##6(s.KT, __VA_ARGS__);      \
    case 7: return FN##7(s.KT, __VA_ARGS__);      \
    case 8: return FN##8(s.KT, __VA_ARGS__);      \
    default: return cudaErrorInvalidValue;        \
  }

cudaError_t launch_em_pass(EmShape s, bool final_sweep, const EmPassArgs& a, int nwork, int F, cudaStream_t st) {
  GSS_M_SWITCH(launch_em_pass_m, final_sweep, a, nwork, F, st)
}
cudaError_t launch_em_update(EmShape s, const EmUpdateArgs& a, int nseg, cudaStream_t st) {
  GSS_M_SWITCH(launch_em_update_m, a, nseg, st)
}
cudaError_t launch_mvdr_stats(EmShape s, const StatsPassArgs& a, int nwork, int F, cudaStream_t st) {
  GSS_M_SWITCH(launch_mvdr_stats_m, a, nwork, F, st)
}
cudaError_t launch_mvdr_stats_final(EmShape s, const StatsFinalArgs& a, int nseg, cudaStream_t st) {
  GSS_M_SWITCH(launch_mvdr_stats_final_m, a, nseg, st)
}

}  // namespace gssb
