// gemm_big_i2.cu -- explicit instantiations of the persistent GEMM (gemm_big_impl.cuh),
// split across units so nvcc compiles them in parallel.
#include "gemm_big_impl.cuh"

namespace srl {
namespace bigk {
#define X(TOK, AMN, BMN, EK) SRL_BIG_INSTANTIATE(TOK, AMN, BMN, EK)
X(128, false, false, 0) X(128, false, false, 1) X(128, false, false, 2) X(128, false, false, 3)
#undef X
}  // namespace bigk
}  // namespace srl
