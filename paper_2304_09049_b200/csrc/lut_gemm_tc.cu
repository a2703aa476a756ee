// lut_gemm_tc.cu — placeholder until the tcgen05 kind::i8 variant lands.
#include "common.cuh"
namespace dg {
bool tc_available() { return false; }
dg_status lut_gemm_tc(const uint8_t *, int64_t, const uint8_t *, int64_t, int64_t, int64_t, int64_t,
                      const int32_t[4], const int32_t[4], void *, int64_t, const RequantArgs *,
                      cudaStream_t) {
    return DG_ERR_UNSUPPORTED;
}
}  // namespace dg
