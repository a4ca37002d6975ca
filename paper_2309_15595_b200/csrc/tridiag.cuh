// tridiag.cuh -- the Hermitian eigensolver of Rayleigh-Ritz (Alg.2 l.20 "HEEVD"; the paper
// calls cuSOLVER xHEEVD) as own GPU kernels, in three stages:
//
//  1. Householder tridiagonalisation (LAPACK xHETD2 order, lower): for j = 0 .. n-2 the reflector
//     H_j = I - tau_j v_j v_j^H of xLARFG annihilates A[j+2:, j] (beta_j real), then
//     p = tau A22 v, w = p - (tau/2)(p^H v) v, A22 -= v w^H + w v^H on the full (both-triangle)
//     trailing matrix.  A = Q T Q^H, Q = H_0 H_1 .. H_{n-2}, T real symmetric tridiagonal (d, e).
//  2. Cuppen divide and conquer on T (LAPACK xSTEDC / xLAED0-3 logic): every off-diagonal torn,
//     T = T^ + sum_i e_i w_i w_i^T (w_i = e_i + e_{i+1}), 1 x 1 leaves, pairs of blocks merged
//     level by level: D + rho z z^T with z = (last row of Q1, first row of Q2) / sqrt(2),
//     rho = 2 e; deflation of tiny z and of close d by Givens rotations (host, xLAED2 rules);
//     the secular equation 1 + rho sum z_i^2 / (d_i - lambda) = 0 by bisection relative to the
//     nearer pole (one thread per root); z recomputed from the roots (Gu-Eisenstat / Loewner,
//     so the eigenvectors are numerically orthogonal); eigenvectors (d_i - lambda)^-1 z^;
//     Q_new = Q(:, kept) U by a batched FP64 GEMM.
//  3. Back-transformation X = Q Z with the reflectors in blocks of 128 (compact WY, xLARFT):
//     Y <- Y - V (T (V^H Y)) on the tensor-core GEMMs.
#pragma once
#include "qr_kernels.cuh"

namespace chase {

constexpr int TRD_THREADS = 1024;

// ---------------------------------------------------------------------------------- stage 1
// Reflector of column j (one CTA): x = A[j+1:n, j]; LAPACK zlarfg(m, alpha, x(2:m)):
//   beta = -sign(Re alpha) ||(alpha, x)||, tau = (beta - alpha) / beta, v = (1, x / (alpha - beta));
//   H = I when x(2:m) = 0 and alpha is real.  Writes v (Vst[:, j], rows j+1.. ; vbuf[0:m]), tau[j],
//   d[j] = Re A[j, j], e[j] = beta.
__global__ void __launch_bounds__(TRD_THREADS)
    trd_reflect_kernel(const double2* A, long long lda, int n, int j, double2* Vst, long long ldv,
                       double2* vbuf, double2* tau, double* d, double* e) {
  __shared__ double red[TRD_THREADS / 32];
  const int m = n - j - 1, tid = threadIdx.x;
  const double2* x = A + (long long)(j + 1) + (long long)j * lda;
  double s = 0.0;
  for (int i = 1 + tid; i < m; i += TRD_THREADS) s += x[i].x * x[i].x + x[i].y * x[i].y;
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((tid & 31) == 0) red[tid >> 5] = s;
  __syncthreads();
  double xn2 = 0.0;
  for (int w = 0; w < TRD_THREADS / 32; ++w) xn2 += red[w];
  const double ar = x[0].x, ai = x[0].y;
  double beta;
  double2 t, inv;
  if (xn2 == 0.0 && ai == 0.0) {
    beta = ar;
    t = make_double2(0.0, 0.0);
    inv = make_double2(1.0, 0.0);
  } else {
    beta = -copysign(sqrt(ar * ar + ai * ai + xn2), ar);
    t = make_double2((beta - ar) / beta, -ai / beta);
    const double dr = ar - beta, di = ai, den = dr * dr + di * di;   // 1 / (alpha - beta)
    inv = make_double2(dr / den, -di / den);
  }
  for (int i = tid; i < m; i += TRD_THREADS) {
    const double2 v = i == 0 ? make_double2(1.0, 0.0) : s_mul(x[i], inv);
    vbuf[i] = v;
    Vst[(long long)(j + 1 + i) + (long long)j * ldv] = v;
  }
  if (tid == 0) {
    tau[j] = t;
    d[j] = A[(long long)j + (long long)j * lda].x;
    e[j] = beta;
    if (j == n - 2) d[n - 1] = A[(long long)(n - 1) + (long long)(n - 1) * lda].x;
  }
}

// p = tau A22 v with A22 = A[j+1:, j+1:] Hermitian: p[c] = tau sum_r conj(A22[r, c]) v[r] (one warp
// per column c, the column read contiguously); CTA partials of p^H v; the last CTA forms
// w = p - (tau/2)(p^H v) v in fixed order (deterministic).
constexpr int TRD_GEMV_WARPS = 8;
__global__ void __launch_bounds__(TRD_GEMV_WARPS * 32)
    trd_gemv_kernel(const double2* A, long long lda, int n, int j, const double2* vbuf,
                    const double2* tau, double2* pbuf, double2* wbuf, double* part, unsigned* ctr) {
  const int m = n - j - 1, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double2 t = tau[j];
  const int c = blockIdx.x * TRD_GEMV_WARPS + warp;
  __shared__ double2 dots[TRD_GEMV_WARPS];
  __shared__ bool last;
  double2 dot = make_double2(0.0, 0.0);
  if (c < m) {
    const double2* col = A + (long long)(j + 1) + (long long)(j + 1 + c) * lda;
    double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0;   // loads in flight together
    int r = lane;
    for (; r + 96 < m; r += 128) {
      a0 = s_add(a0, s_cmul(col[r], vbuf[r]));                         // conj(a) v
      a1 = s_add(a1, s_cmul(col[r + 32], vbuf[r + 32]));
      a2 = s_add(a2, s_cmul(col[r + 64], vbuf[r + 64]));
      a3 = s_add(a3, s_cmul(col[r + 96], vbuf[r + 96]));
    }
    for (; r < m; r += 32) a0 = s_add(a0, s_cmul(col[r], vbuf[r]));
    double2 acc = s_add(s_add(a0, a1), s_add(a2, a3));
    for (int o = 16; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    const double2 p = s_mul(t, acc);
    if (lane == 0) pbuf[c] = p;
    dot = s_cmul(p, vbuf[c]);                          // conj(p_c) v_c
  }
  if (lane == 0) dots[warp] = dot;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 s = make_double2(0.0, 0.0);
    for (int w = 0; w < TRD_GEMV_WARPS; ++w) s = s_add(s, dots[w]);
    part[2 * blockIdx.x] = s.x;
    part[2 * blockIdx.x + 1] = s.y;
    __threadfence();
    last = atomicAdd(ctr, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // fixed-order total of the CTA partials with all threads: thread q sums b = q, q + 256, ...,
  // then a shared-memory tree over the 256 thread sums
  __shared__ double2 tsum[TRD_GEMV_WARPS * 32];
  __shared__ double2 alpha;
  {
    double2 s = make_double2(0.0, 0.0);
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
      s = s_add(s, make_double2(__ldcg(part + 2 * b), __ldcg(part + 2 * b + 1)));
    tsum[threadIdx.x] = s;
  }
  __syncthreads();
  for (int w = TRD_GEMV_WARPS * 16; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) tsum[threadIdx.x] = s_add(tsum[threadIdx.x], tsum[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    // alpha = -(1/2) tau (p^H v)   (xHETD2)
    const double2 a = s_mul(t, tsum[0]);
    alpha = make_double2(-0.5 * a.x, -0.5 * a.y);
    *ctr = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) wbuf[i] = s_add(__ldcg(pbuf + i), s_mul(alpha, vbuf[i]));
}

// A22 -= v w^H + w v^H (both triangles; 32 x 32 tiles, coalesced along rows)
__global__ void __launch_bounds__(256)
    trd_rank2_kernel(double2* A, long long lda, int n, int j, const double2* vbuf, const double2* wbuf) {
  const int m = n - j - 1;
  const int r = blockIdx.x * 32 + (threadIdx.x & 31);
  if (r >= m) return;
  const double2 vr = vbuf[r], wr = wbuf[r];
  for (int c = blockIdx.y * 32 + (threadIdx.x >> 5); c < min(m, blockIdx.y * 32 + 32); c += 8) {
    double2* a = A + (long long)(j + 1 + r) + (long long)(j + 1 + c) * lda;
    const double2 vc = vbuf[c], wc = wbuf[c];
    // v_r conj(w_c) + w_r conj(v_c)
    const double2 u = s_add(s_mul(vr, make_double2(wc.x, -wc.y)), s_mul(wr, make_double2(vc.x, -vc.y)));
    *a = s_sub(*a, u);
  }
}

// ---- fused pipeline (two launches per column instead of three):
//  trd_next_reflect_kernel(j): column j+1 of A22_j updated by step j's rank 2 (v_j, w_j), then the
//     reflector of column j+1 from it (as trd_reflect_kernel), d[j+1] = Re A[j+1, j+1];
//  trd_fused_kernel(j): the rest of step j's rank-2 update restricted to A22_{j+1} = A[j+2:, j+2:]
//     (the only part read again), fused with step j+1's GEMV p' = tau' A22_{j+1} v' and w' -- one
//     read and one write of the trailing matrix per column instead of two reads and one write.
__global__ void __launch_bounds__(TRD_THREADS)
    trd_next_reflect_kernel(const double2* A, long long lda, int n, int j, const double2* v,
                            const double2* w, double2* Vst, long long ldv, double2* vnext,
                            double2* tau, double* d, double* e) {
  __shared__ double red[TRD_THREADS / 32];
  __shared__ double2 head[2];
  const int m = n - j - 1, tid = threadIdx.x;            // A22_j is m x m; next column = its col 0
  const double2 w0 = w[0], v0 = v[0];
  const double2 cw0 = make_double2(w0.x, -w0.y), cv0 = make_double2(v0.x, -v0.y);
  const double2* col = A + (long long)(j + 1) + (long long)(j + 1) * lda;   // A22_j[:, 0]
  auto upd = [&](int r) {                                 // updated A22_j[r, 0]
    return s_sub(col[r], s_add(s_mul(v[r], cw0), s_mul(w[r], cv0)));
  };
  double s = 0.0;
  for (int r = 2 + tid; r < m; r += TRD_THREADS) {
    const double2 x = upd(r);
    s += x.x * x.x + x.y * x.y;
  }
  if (tid == 0) {
    head[0] = upd(0);
    head[1] = m > 1 ? upd(1) : make_double2(0.0, 0.0);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((tid & 31) == 0) red[tid >> 5] = s;
  __syncthreads();
  double xn2 = 0.0;
  for (int q = 0; q < TRD_THREADS / 32; ++q) xn2 += red[q];
  const int jn = j + 1, mn = m - 1;                       // next column index, its length
  const double ar = head[1].x, ai = head[1].y;
  double beta;
  double2 t, inv;
  if (xn2 == 0.0 && ai == 0.0) {
    beta = ar;
    t = make_double2(0.0, 0.0);
    inv = make_double2(1.0, 0.0);
  } else {
    beta = -copysign(sqrt(ar * ar + ai * ai + xn2), ar);
    t = make_double2((beta - ar) / beta, -ai / beta);
    const double dr = ar - beta, di = ai, den = dr * dr + di * di;
    inv = make_double2(dr / den, -di / den);
  }
  for (int i = tid; i < mn; i += TRD_THREADS) {
    const double2 vv = i == 0 ? make_double2(1.0, 0.0) : s_mul(upd(i + 1), inv);
    vnext[i] = vv;
    Vst[(long long)(jn + 1 + i) + (long long)jn * ldv] = vv;
  }
  if (tid == 0) {
    tau[jn] = t;
    d[jn] = head[0].x;
    e[jn] = beta;
  }
}

constexpr int TRD_FUSED_WARPS = 8;
__global__ void __launch_bounds__(TRD_FUSED_WARPS * 32)
    trd_fused_kernel(double2* __restrict__ A, long long lda, int n, int j, const double2* __restrict__ v,
                     const double2* __restrict__ w, const double2* __restrict__ vn, const double2* tau,
                     double2* pbuf, double2* wbuf, double* part, unsigned* ctr) {
  const int m = n - j - 1, mn = m - 1, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double2 tn = tau[j + 1];
  const int c = blockIdx.x * TRD_FUSED_WARPS + warp;     // column of A22_{j+1}
  __shared__ double2 dots[TRD_FUSED_WARPS];
  __shared__ bool last;
  double2 dot = make_double2(0.0, 0.0);
  if (c < mn) {
    // A22_j[r, c+1] for r = 1..m-1  ->  A22_{j+1}[r-1, c]
    double2* __restrict__ colp = A + (long long)(j + 2) + (long long)(j + 2 + c) * lda;
    const double2 wc = w[c + 1], vc = v[c + 1];
    const double2 cwc = make_double2(wc.x, -wc.y), cvc = make_double2(vc.x, -vc.y);
    double2 a0 = make_double2(0.0, 0.0), a1 = a0;
    int r = lane;
    for (; r + 96 < mn; r += 128) {                       // 4 columns chunks, loads first
      double2 x[4], y[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) x[q] = colp[r + 32 * q];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        y[q] = s_sub(x[q], s_add(s_mul(v[r + 32 * q + 1], cwc), s_mul(w[r + 32 * q + 1], cvc)));
        colp[r + 32 * q] = y[q];
      }
      a0 = s_add(a0, s_add(s_cmul(y[0], vn[r]), s_cmul(y[2], vn[r + 64])));
      a1 = s_add(a1, s_add(s_cmul(y[1], vn[r + 32]), s_cmul(y[3], vn[r + 96])));
    }
    for (; r < mn; r += 32) {
      const double2 y = s_sub(colp[r], s_add(s_mul(v[r + 1], cwc), s_mul(w[r + 1], cvc)));
      colp[r] = y;
      a0 = s_add(a0, s_cmul(y, vn[r]));
    }
    double2 acc = s_add(a0, a1);
    for (int o = 16; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    const double2 p = s_mul(tn, acc);
    if (lane == 0) pbuf[c] = p;
    dot = s_cmul(p, vn[c]);
  }
  if (lane == 0) dots[warp] = dot;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 s = make_double2(0.0, 0.0);
    for (int q = 0; q < TRD_FUSED_WARPS; ++q) s = s_add(s, dots[q]);
    part[2 * blockIdx.x] = s.x;
    part[2 * blockIdx.x + 1] = s.y;
    __threadfence();
    last = atomicAdd(ctr, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double2 tsum[TRD_FUSED_WARPS * 32];
  __shared__ double2 alpha;
  {
    double2 s = make_double2(0.0, 0.0);
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
      s = s_add(s, make_double2(__ldcg(part + 2 * b), __ldcg(part + 2 * b + 1)));
    tsum[threadIdx.x] = s;
  }
  __syncthreads();
  for (int q = TRD_FUSED_WARPS * 16; q > 0; q >>= 1) {
    if ((int)threadIdx.x < q) tsum[threadIdx.x] = s_add(tsum[threadIdx.x], tsum[threadIdx.x + q]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double2 a = s_mul(tn, tsum[0]);
    alpha = make_double2(-0.5 * a.x, -0.5 * a.y);
    *ctr = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < mn; i += blockDim.x) wbuf[i] = s_add(__ldcg(pbuf + i), s_mul(alpha, vn[i]));
}

__global__ void trd_last_diag_kernel(const double2* A, long long lda, int n, double* d) {
  d[n - 1] = A[(long long)(n - 1) + (long long)(n - 1) * lda].x;
}

// A <- (A + A^H) / 2 (the reduced quotient B2^H B is Hermitian only up to rounding)
__global__ void trd_symmetrize_kernel(double2* A, long long lda, int n) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)n * n) return;
  const int r = (int)(idx % n), c = (int)(idx / n);
  if (r > c) return;
  double2* a = A + r + (long long)c * lda;
  double2* b = A + c + (long long)r * lda;
  if (r == c) {
    a->y = 0.0;
    return;
  }
  const double2 x = *a, y = *b;
  const double2 m = make_double2(0.5 * (x.x + y.x), 0.5 * (x.y - y.y));
  *a = m;
  *b = make_double2(m.x, -m.y);
}

// ---------------------------------------------------------------------------------- stage 2
// Z (n x n, ld n, real) <- I; dd[i] = d[i] - e[i-1] - e[i] (every off-diagonal torn)
__global__ void dc_init_kernel(const double* d, const double* e, int n, double* dd, double* Z) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < (long long)n * n) Z[idx] = (idx % n) == (idx / n) ? 1.0 : 0.0;
  if (idx < n) {
    const int i = (int)idx;
    double v = d[i];
    if (i > 0) v -= e[i - 1];
    if (i < n - 1) v -= e[i];
    dd[i] = v;
  }
}

// Merge descriptor of one level (packed arrays; all indices block-local unless noted).
struct DcMerge {
  int s, k;            // block rows/cols [s, s+k) of Z
  int k1;              // rows of the first child
  int kk;              // non-deflated roots
  int off;             // offset of this merge in the packed K/dK/zK/roots arrays (== s)
  int nrot, roff;      // Givens rotations (count, offset in the rotation arrays)
  int flip;            // the problem was negated (rho < 0)
  double rho;          // > 0
  long long uoff;      // offset of U (kk x kk, ld kk) in the U buffer
};

// z = (last row of Q1 restricted to Q1's columns, first row of Q2 restricted to Q2's columns)
__global__ void dc_gather_z_kernel(const double* Z, int n, const DcMerge* M, int nm, double* z) {
  const int mi = blockIdx.y;
  if (mi >= nm) return;
  const DcMerge mg = M[mi];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= mg.k) return;
  const int row = i < mg.k1 ? mg.s + mg.k1 - 1 : mg.s + mg.k1;
  z[mg.s + i] = Z[(long long)row + (long long)(mg.s + i) * n];
}

// Givens rotations of the deflation, in order, on the block's rows (thread per row):
// (x, y) <- (c x + s y, c y - s x) for columns (a, b) (xLAED2's DROT)
__global__ void dc_rotate_kernel(double* Z, int n, const DcMerge* M, int nm, const int* ra,
                                 const int* rb, const double* rc, const double* rs) {
  const int mi = blockIdx.y;
  if (mi >= nm) return;
  const DcMerge mg = M[mi];
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= mg.k || mg.nrot == 0) return;
  double* row = Z + (long long)(mg.s + r);
  for (int q = 0; q < mg.nrot; ++q) {
    const int a = mg.s + ra[mg.roff + q], b = mg.s + rb[mg.roff + q];
    const double c = rc[mg.roff + q], s = rs[mg.roff + q];
    const double x = row[(long long)a * n], y = row[(long long)b * n];
    row[(long long)a * n] = c * x + s * y;
    row[(long long)b * n] = c * y - s * x;
  }
}

// Secular roots: one warp per (merge, root m), the lanes splitting the sums over i (fixed order:
// lane partials, then a butterfly).  dK ascending, rho > 0; root m lies in (dK[m], dK[m+1]) (the
// last in (dK[kk-1], dK[kk-1] + rho z^T z)).  Bisection on tau relative to the nearer pole
// (origin org[m]), so d_i - lambda = (dK[i] - dK[org]) - tau keeps its digits.
__global__ void dc_secular_kernel(const DcMerge* M, int nm, const double* dK, const double* zK,
                                  int* org, double* tau, double* lam) {
  const int mi = blockIdx.y;
  if (mi >= nm) return;
  const DcMerge mg = M[mi];
  const int lane = threadIdx.x & 31;
  const int mroot = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (mroot >= mg.kk) return;
  const double* d = dK + mg.off;
  const double* z = zK + mg.off;
  const int kk = mg.kk;
  const double rho = mg.rho;
  auto wsum = [&](double x) {
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
  };
  double zz = 0.0;
  for (int i = lane; i < kk; i += 32) zz += z[i] * z[i];
  zz = wsum(zz);
  const double lo_pole = d[mroot];
  const double hi_pole = mroot + 1 < kk ? d[mroot + 1] : d[kk - 1] + rho * zz;
  auto f_at = [&](int o, double t) {                 // f(d[o] + t), same value in every lane
    double sacc = 0.0;
    const double dor = d[o];
    for (int i = lane; i < kk; i += 32) sacc += z[i] * z[i] / ((d[i] - dor) - t);
    return 1.0 + rho * wsum(sacc);
  };
  int o = mroot;
  double a, b;                                       // tau interval, f(a) < 0 < f(b)
  const double mid = 0.5 * (hi_pole - lo_pole);
  if (mroot + 1 < kk && f_at(mroot, mid) < 0.0) {    // root in (mid, hi): origin = upper pole
    o = mroot + 1;
    a = -mid;
    b = 0.0;
  } else {
    a = 0.0;
    b = mroot + 1 < kk ? mid : hi_pole - lo_pole;
  }
  for (int it = 0; it < 200; ++it) {                 // warp-uniform control flow
    const double t = 0.5 * (a + b);
    if (t == a || t == b) break;
    const double f = f_at(o, t);
    if (f < 0.0) a = t;
    else if (f > 0.0) b = t;
    else { a = b = t; break; }
  }
  if (lane == 0) {
    const double t = 0.5 * (a + b);
    org[mg.off + mroot] = o;
    tau[mg.off + mroot] = t;
    lam[mg.off + mroot] = d[o] + t;
  }
}

// Gu-Eisenstat: z^_i = sign(z_i) sqrt( (lam_{kk-1} - d_i)/rho prod_{m<i} (lam_m - d_i)/(d_m - d_i)
//                                      prod_{i<=m<kk-1} (lam_m - d_i)/(d_{m+1} - d_i) )
// with lam_m - d_i = (d[org_m] - d_i) + tau_m (all ratios positive and bounded).
__global__ void dc_zhat_kernel(const DcMerge* M, int nm, const double* dK, const double* zK,
                               const int* org, const double* tau, double* zh) {
  const int mi = blockIdx.y;
  if (mi >= nm) return;
  const DcMerge mg = M[mi];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= mg.kk) return;
  const double* d = dK + mg.off;
  const int* og = org + mg.off;
  const double* tu = tau + mg.off;
  const int kk = mg.kk;
  const double di = d[i];
  double p = ((d[og[kk - 1]] - di) + tu[kk - 1]) / mg.rho;
  for (int m = 0; m < kk - 1; ++m) {
    const double num = (d[og[m]] - di) + tu[m];
    const double den = m < i ? d[m] - di : d[m + 1] - di;
    p *= num / den;
  }
  zh[mg.off + i] = copysign(sqrt(fabs(p)), zK[mg.off + i]);
}

// U[:, m] = (z^_i / (d_i - lam_m))_i / norm  (one warp per root m; U kk x kk, ld kk)
__global__ void dc_vectors_kernel(const DcMerge* M, int nm, const double* dK, const double* zh,
                                  const int* org, const double* tau, double* U) {
  const int mi = blockIdx.y;
  if (mi >= nm) return;
  const DcMerge mg = M[mi];
  const int lane = threadIdx.x & 31;
  const int mroot = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (mroot >= mg.kk) return;
  const double* d = dK + mg.off;
  const int o = org[mg.off + mroot];
  const double t = tau[mg.off + mroot];
  double* u = U + mg.uoff + (long long)mroot * mg.kk;
  double s = 0.0;
  for (int i = lane; i < mg.kk; i += 32) {
    const double v = zh[mg.off + i] / ((d[i] - d[o]) - t);
    u[i] = v;
    s += v * v;
  }
  for (int x = 16; x > 0; x >>= 1) s += __shfl_xor_sync(0xffffffffu, s, x);
  const double inv = 1.0 / sqrt(s);
  for (int i = lane; i < mg.kk; i += 32) u[i] *= inv;
}

// Z2[block rows, s + m] = sum_i Z[block rows, s + Kidx[i]] U[i, m]  (m < kk), batched FP64 GEMM:
// 64 x 64 output tiles, 256 threads with 4 x 4 outputs each, k in chunks of 16 through smem.
__global__ void __launch_bounds__(256)
    dc_gemm_kernel(const double* Z, double* Z2, int n, const DcMerge* M, const int* Kidx,
                   const double* U) {
  const DcMerge mg = M[blockIdx.z];
  const int r0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
  if (r0 >= mg.k || c0 >= mg.kk) return;
  __shared__ double As[16][65], Bs[16][65];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  const int* K = Kidx + mg.off;
  const double* Ub = U + mg.uoff;
  for (int k0 = 0; k0 < mg.kk; k0 += 16) {
      for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int kk_ = e / 64, rr = e % 64;            // A: rows r0+rr, column K[k0+kk_]
      const int kc = k0 + kk_;
      As[kk_][rr] = (kc < mg.kk && r0 + rr < mg.k) ? Z[(long long)(mg.s + r0 + rr) + (long long)(mg.s + K[kc]) * n] : 0.0;
      const int kq = e % 16, cc = e / 16;             // B: U[k0+kq, c0+cc], k fastest (coalesced)
      Bs[kq][cc] = (k0 + kq < mg.kk && c0 + cc < mg.kk) ? Ub[(long long)(k0 + kq) + (long long)(c0 + cc) * mg.kk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      double a[4], b[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) a[x] = As[q][tx + 16 * x];
#pragma unroll
      for (int y = 0; y < 4; ++y) b[y] = Bs[q][ty + 16 * y];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] += a[x] * b[y];
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int r = r0 + tx + 16 * x, c = c0 + ty + 16 * y;
      if (r < mg.k && c < mg.kk) Z2[(long long)(mg.s + r) + (long long)(mg.s + c) * n] = acc[x][y];
    }
}

// deflated columns (and whole unmerged blocks): Z2[block rows, s + dst] = Z[block rows, s + src]
__global__ void dc_copy_cols_kernel(const double* Z, double* Z2, int n, const DcMerge* M,
                                    const int* src, const int* dst, const int* coff, const int* ccnt) {
  const DcMerge mg = M[blockIdx.z];
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= mg.k) return;
  for (int q = blockIdx.y; q < ccnt[blockIdx.z]; q += gridDim.y) {
    const int a = src[coff[blockIdx.z] + q], b = dst[coff[blockIdx.z] + q];
    Z2[(long long)(mg.s + r) + (long long)(mg.s + b) * n] = Z[(long long)(mg.s + r) + (long long)(mg.s + a) * n];
  }
}

// Y (complex, ld ldy) <- Z (real, ld n)
__global__ void dc_to_complex_kernel(const double* Z, int n, double2* Y, long long ldy) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)n * n) return;
  const long long r = idx % n, c = idx / n;
  Y[r + c * ldy] = make_double2(Z[idx], 0.0);
}

}  // namespace chase
