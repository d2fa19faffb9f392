// ctc_pair.cu -- launches of the alpha || beta pair kernel (ctc_pair_kernel.cuh)
// for K = 1..6 label pairs per chain thread; K = 8 lives in ctc_pair_k8.cu.
#include "ctc_pair_kernel.cuh"

namespace ds2ctc {

#ifdef DS2CTC_EPOCH_TIMING
extern "C" int ds2ctc_debug_epoch_clocks(long long* host) {
  return cudaMemcpyFromSymbol(host, g_epoch_clock, sizeof(g_epoch_clock));
}
extern "C" int ds2ctc_debug_meet_clocks(long long* host) {
  int e = cudaMemcpyFromSymbol(host, g_meet_clock, sizeof(g_meet_clock));
  if (e) return e;
  return cudaMemcpyFromSymbol(host + 16, g_kernel_end, sizeof(g_kernel_end));
}
extern "C" int ds2ctc_debug_prologue_clocks(long long* host) {
  return cudaMemcpyFromSymbol(host, g_pro_clock, sizeof(g_pro_clock));
}
extern "C" int ds2ctc_debug_step_clocks(long long* host) {
  return cudaMemcpyFromSymbol(host, g_step_clock, sizeof(g_step_clock));
}
#endif

int read_watchdog(unsigned long long* out4) {
  // the first record of either translation unit (K = 1..6 here, K = 8 in ctc_pair_k8.cu)
  int e = read_watchdog_tu(out4);
  if (e != cudaSuccess) return e;
  unsigned long long k8[4];
  e = read_watchdog_k8(k8);
  if (e != cudaSuccess) return e;
  if (out4[0] == 0)
    for (int i = 0; i < 4; ++i) out4[i] = k8[i];
  return cudaSuccess;
}

int launch_pair(const PairArgs& a, void* stream) {
  if (a.B == 0) return cudaSuccess;
  if (a.g.dual) {
    switch (a.g.K) {
      case 1: return launch_k<1, 2>(a, stream);
      case 2: return launch_k<2, 2>(a, stream);
      case 3: return launch_k<3, 2>(a, stream);
      case 4: return launch_k<4, 2>(a, stream);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (a.g.K) {
    case 1: return launch_k<1>(a, stream);
    case 2: return launch_k<2>(a, stream);
    case 3: return launch_k<3>(a, stream);
    case 4: return launch_k<4>(a, stream);
    case 6: return launch_k<6>(a, stream);
    case 8: return launch_pair_k8(a, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ds2ctc
