#include <cuda_runtime.h>
#include "/root/repo/paper_1512_02595_b200/csrc/ds2ctc_internal.h"
namespace ds2ctc {
int launch_pair(const PairArgs&, void*) { return 0; }
int launch_dense(const PairArgs&, bool, void*) { return 0; }
int launch_finalize(const PairArgs&, void*) { return 0; }
int launch_loss_sum(const float*, int, double*, void*) { return 0; }
int read_watchdog(unsigned long long*) { return 0; }
}
