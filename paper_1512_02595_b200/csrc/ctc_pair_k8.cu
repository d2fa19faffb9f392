// ctc_pair_k8.cu -- the K = 8 instantiation of the pair kernel (labels longer
// than 671 symbols: up to ten chain warps, 384 threads, 168 registers). Built
// with ptxas -O1 (paper_1512_02595_b200/build.py): ptxas 12.9 -O3 segfaults on
// this instantiation of the slot-major column code at that register budget.
#include "ctc_pair_kernel.cuh"

namespace ds2ctc {

int launch_pair_k8(const PairArgs& a, void* stream) { return launch_k<8>(a, stream); }

int read_watchdog_k8(unsigned long long* out4) { return read_watchdog_tu(out4); }

}  // namespace ds2ctc
