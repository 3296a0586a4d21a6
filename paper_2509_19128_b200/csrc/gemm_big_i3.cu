// gemm_big_i3.cu -- explicit instantiations of the persistent GEMM (gemm_big_impl.cuh),
// split across units so nvcc compiles them in parallel.
#include "gemm_big_impl.cuh"

namespace srl {
namespace bigk {
#define X(TOK, AMN, BMN, EK) SRL_BIG_INSTANTIATE(TOK, AMN, BMN, EK)
X(128, false, false, 4) X(128, false, false, 5) X(128, false, false, 6) X(128, false, false, 7)
#undef X
}  // namespace bigk
}  // namespace srl
