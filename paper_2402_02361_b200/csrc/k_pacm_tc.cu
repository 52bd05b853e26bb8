// k_pacm_tc.cu — tcgen05/TMEM PaCM (placeholder until the tensor-core
// kernel lands; the fp64 path serves every precision request meanwhile).
#include "tt_kernels.h"

namespace tt {

bool pacm_tc_supported(const DevSketch&, int) { return false; }
size_t pacm_tc_packed_bytes(int) { return 16; }
int launch_pacm_tc_pack(const double*, int, void*, cudaStream_t) { return -1; }
int launch_pacm_tc(const DevSketch&, const DevDevice&, CandRef, const int64_t*, int64_t, const void*, int, double*,
                   cudaStream_t) {
  return -1;
}

}  // namespace tt
