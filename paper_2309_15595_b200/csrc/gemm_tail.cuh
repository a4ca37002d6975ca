// gemm_tail.cuh -- wave-quantisation tail of the big GEMMs (the filter HEMM steps).
//
// A step's output has T = m_tiles x n_tiles tiles, one CTA per SM at a time, all of equal cost;
// when T is not a multiple of the SM count the last wave runs partly empty (C2: T = 11045 on
// 148 SMs = 74.6 waves, the last 89 CTAs leave 59 SMs idle for a whole wave, 0.5 % of the step).
// The host launches the plain GEMM on the first T_main tiles of the raster and the remaining
// T_tail tiles as a split-K launch (zgemm/dgemm SPLIT variant, tail_tiles > 0: S copies of the
// tail, copy s summing its own K range into a tile-local partial); this kernel then sums the S
// partials of every tail tile in fixed order and applies the same epilogue as the plain GEMM
// (band shift, alpha, beta * old), so the result differs from the one-launch GEMM only in the
// order of the K summation.
#pragma once
#include "common.cuh"

namespace chase {

__device__ __forceinline__ double2 tl_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double tl_add(double a, double b) { return a + b; }
__device__ __forceinline__ double2 tl_axpy(double2 acc, double c, double2 x) {   // acc - c x
  return make_double2(acc.x - c * x.x, acc.y - c * x.y);
}
__device__ __forceinline__ double tl_axpy(double acc, double c, double x) { return acc - c * x; }
__device__ __forceinline__ double2 tl_scale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double tl_scale(double a, double s) { return a * s; }
__device__ __forceinline__ double2 tl_fma(double2 acc, double b, double2 o) {   // acc + b o
  return make_double2(acc.x + b * o.x, acc.y + b * o.y);
}
__device__ __forceinline__ double tl_fma(double acc, double b, double o) { return acc + b * o; }

struct TailArgs {
  int S, tail_tiles, tile_offset, M, N;
  long long ldo, ldx;
  double alpha, beta, c;
  int use_beta, band_lo, band_hi, band_shift;
  const int* band_map;
};

// one CTA per tail tile; the raster (tile -> (m0, n0)) is the GEMM's grouped rasterisation
template <typename T, int BM, int BN, int GROUP_M>
__global__ void __launch_bounds__(256)
    gemm_tail_epilogue_kernel(const T* __restrict__ part, T* out, const T* xin, const TailArgs a) {
  const int j = blockIdx.x;
  const int t = a.tile_offset + j;
  const int n_tiles = (a.N + BN - 1) / BN, m_tiles = (a.M + BM - 1) / BM;
  const int group = t / (GROUP_M * n_tiles);
  const int first_m = group * GROUP_M;
  const int gm = min(GROUP_M, m_tiles - first_m);
  const int within = t - group * GROUP_M * n_tiles;
  const int m0 = (first_m + within % gm) * BM, n0 = (within / gm) * BN;
  for (int e = threadIdx.x; e < BM * BN; e += blockDim.x) {
    const int row = m0 + (e % BM), col = n0 + (e / BM);
    if (row >= a.M || col >= a.N) continue;
    T acc = part[(long long)j * (BM * BN) + e];
    for (int s = 1; s < a.S; ++s)
      acc = tl_add(acc, part[((long long)s * a.tail_tiles + j) * (BM * BN) + e]);
    const int bsrc = a.band_map != nullptr ? a.band_map[row]
                     : (row >= a.band_lo && row < a.band_hi ? row + a.band_shift : -1);
    if (bsrc >= 0) acc = tl_axpy(acc, a.c, xin[(long long)bsrc + (long long)col * a.ldx]);
    acc = tl_scale(acc, a.alpha);
    T* o = out + (long long)row + (long long)col * a.ldo;
    if (a.use_beta) acc = tl_fma(acc, a.beta, *o);
    *o = acc;
  }
}

}  // namespace chase
