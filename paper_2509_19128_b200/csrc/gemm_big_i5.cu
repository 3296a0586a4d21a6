// gemm_big_i5.cu -- explicit instantiations of the persistent GEMM (gemm_big_impl.cuh),
// split across units so nvcc compiles them in parallel.
#include "gemm_big_impl.cuh"

namespace srl {
namespace bigk {
#define X(TOK, AMN, BMN, EK) SRL_BIG_INSTANTIATE(TOK, AMN, BMN, EK)
X(256, true, false, 0) X(256, true, false, 6) X(256, true, false, 8) X(128, true, false, 0) X(128, true, false, 6) X(128, true, false, 8)
#undef X
}  // namespace bigk
}  // namespace srl
