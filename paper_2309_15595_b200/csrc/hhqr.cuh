// hhqr.cuh -- the Householder QR fallback of Alg.4 l.8-9 (the paper calls
// ScaLAPACK's HHQR on the 1D row distribution of the column communicator) as GPU kernels:
// blocked right-looking Householder QR (LAPACK xGEQRF order) with 128-wide panels (the paper's
// ScaLAPACK run used 32; 128 fills the GEMMs' 128-row tiles), then the explicit thin Q
// (xUNGQR order), both distributed over the rows of the column communicator.  The flop-heavy
// pieces (trailing updates with the compact-WY form I - V T V^H, the blocked Q formation) run
// on the tensor-core GEMMs, the V^H (.) products split over K; the latency-bound panel runs
// column by column in the kernels below (the panel stays L2-resident).
//
// Rows are taken in the "virtual" order rank 0's local rows, rank 1's, ... of the column
// communicator (voff = first virtual row of this rank).  For the block distribution this is the
// global order; for block-cyclic it is a row permutation P, and the Q of PX with positive
// diag(R) is PQ -- the same Q (reading #33).
//
// Reflectors follow LAPACK xLARFG: H^H (alpha; x) = (beta; 0), H = I - tau v v^H, v = (1; x /
// (alpha - beta)), beta = -sign(Re alpha) ||(alpha; x)|| real.  Column j of Q is finally scaled
// by sign(beta_j) so diag(R) is non-negative (the CholeskyQR convention).
//
// Grid-wide sums (column norms, v^H C) are per-CTA partials reduced in fixed order by the last
// CTA to finish (deterministic: the q replicas of each column communicator stay bit-identical).
#pragma once
#include "qr_kernels.cuh"

namespace chase {

constexpr int HH_NB = 128;         // panel width (the trailing-update GEMMs get M = 128 tiles)
constexpr int HH_CH = 32;          // panel columns per CTA in the column kernels (blockIdx.y)
constexpr int HH_NCH = HH_NB / HH_CH;
constexpr int HH_THREADS = 256;
constexpr int HH_GRID_MAX = 148;   // row CTAs of the column kernels

__device__ __forceinline__ double2 s_conj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double s_conj(double a) { return a; }
template <typename T> __device__ __forceinline__ T s_make(double re, double im);
template <> __device__ __forceinline__ double2 s_make<double2>(double re, double im) { return make_double2(re, im); }
template <> __device__ __forceinline__ double s_make<double>(double re, double) { return re; }
__device__ __forceinline__ double s_im(double2 a) { return a.y; }
__device__ __forceinline__ double s_im(double) { return 0.0; }
template <typename T> __host__ __device__ constexpr int s_words() { return (int)(sizeof(T) / sizeof(double)); }
__device__ __forceinline__ void s_put(double* d, double2 a) { d[0] = a.x; d[1] = a.y; }
__device__ __forceinline__ void s_put(double* d, double a) { d[0] = a; }

// Sum NV per-thread doubles over the CTA (fixed order: warp butterflies, then warps 0..7) and
// store the CTA total at part[blockIdx.x * NV + k].  Returns true in every thread of the last CTA
// to arrive, which then owns the fixed-order grid-wide sum.
template <int NV>
__device__ bool hh_cta_partial(const double (&v)[NV], double* part, unsigned* ctr) {
  __shared__ double wsum[HH_THREADS / 32][NV];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double x = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) wsum[warp][k] = x;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < NV; k += HH_THREADS) {
    double x = 0.0;
#pragma unroll
    for (int w = 0; w < HH_THREADS / 32; ++w) x += wsum[w][k];
    part[(size_t)blockIdx.x * NV + k] = x;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// fixed-order sum over the CTA partials (last CTA only); resets the arrival counter
template <int NV>
__device__ void hh_grid_total(const double* part, int nv, double* out, unsigned* ctr) {
  for (int k = threadIdx.x; k < nv; k += HH_THREADS) {
    double x = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) x += __ldcg(part + (size_t)b * NV + k);
    out[k] = x;
  }
  if (threadIdx.x == 0) *ctr = 0;
}

// red[0] = sum |X[g, j]|^2 over virtual rows g > j; red[1], red[2] = X[j, j] (re, im) -- the
// pivot's owner contributes it, everyone else 0, so the AllReduce returns it exactly.
template <typename T>
__global__ void __launch_bounds__(HH_THREADS)
    hh_norm_kernel(const T* X, long long ldx, int n_r, long long voff, int j, double* part,
                   double* red, unsigned* ctr) {
  double v[3] = {0.0, 0.0, 0.0};
  const T* col = X + (long long)j * ldx;
  for (int l = blockIdx.x * HH_THREADS + threadIdx.x; l < n_r; l += gridDim.x * HH_THREADS) {
    const long long g = voff + l;
    const T x = col[l];
    if (g > j) v[0] += s_abs2(x);
    else if (g == j) { v[1] = s_re(x); v[2] = s_im(x); }
  }
  if (hh_cta_partial<3>(v, part, ctr)) hh_grid_total<3>(part, 3, red, ctr);
}

// beta, tau and 1/(alpha - beta) of xLARFG from the reduced (||x||^2, alpha)
template <typename T>
__device__ __forceinline__ void hh_reflector(const double* red, double* beta, T* tau, T* inv) {
  const double xn2 = red[0], ar = red[1], ai = red[2];
  if (xn2 == 0.0 && ai == 0.0) {              // H = I
    *beta = ar;
    *tau = s_real<T>(0.0);
    *inv = s_real<T>(1.0);
    return;
  }
  const double b = -copysign(sqrt(ar * ar + ai * ai + xn2), ar);
  *beta = b;
  *tau = s_make<T>((b - ar) / b, -ai / b);
  // 1 / (alpha - beta), alpha - beta = (ar - b) + i ai
  const double dr = ar - b, di = ai, den = dr * dr + di * di;
  *inv = s_make<T>(dr / den, -di / den);
}

// Column j of the panel [.., pend): form v_j into Vp[:, jj] (zeros above the pivot, 1 at it)
// and reduce w = v^H X[:, j+1:pend] -- CTA (r, ch) covers row slice r and the 32 panel columns
// j+1+32ch ..; X[:, j] itself is rewritten only by hh_store_panel_kernel (the CTAs of the other
// chunks still read it).  Chunk ch's last CTA stores w[32ch ..] (red_w).
template <typename T>
__global__ void __launch_bounds__(HH_THREADS)
    hh_reflect_kernel(const T* X, long long ldx, int n_r, long long voff, int j, int pend, T* Vp,
                      long long ldvp, int jj, const double* red_n, double* part, T* red_w,
                      unsigned* ctr, T* tau_out, double* beta_out) {
  constexpr int W = s_words<T>();
  constexpr int NV = HH_CH * W;
  double beta;
  T tau, inv;
  hh_reflector<T>(red_n, &beta, &tau, &inv);
  const int ch = blockIdx.y;
  const int nw = pend - j - 1, c0 = j + 1 + ch * HH_CH;
  const int nc = min(HH_CH, nw - ch * HH_CH);          // columns of this chunk (may be <= 0)
  if (blockIdx.x == 0 && ch == 0 && threadIdx.x == 0) {
    tau_out[j] = tau;
    beta_out[j] = beta;
  }
  T acc[HH_CH];
#pragma unroll
  for (int c = 0; c < HH_CH; ++c) acc[c] = s_real<T>(0.0);
  const T* colj = X + (long long)j * ldx;
  T* vpc = Vp + (long long)jj * ldvp;
  for (int l = blockIdx.x * HH_THREADS + threadIdx.x; l < n_r; l += gridDim.x * HH_THREADS) {
    const long long g = voff + l;
    if (g < j) {
      if (ch == 0) vpc[l] = s_real<T>(0.0);
      continue;
    }
    const T v = g == j ? s_real<T>(1.0) : s_mul(colj[l], inv);
    if (ch == 0) vpc[l] = v;
#pragma unroll
    for (int c = 0; c < HH_CH; ++c)
      if (c < nc) acc[c] = s_add(acc[c], s_cmul(v, X[(long long)l + (long long)(c0 + c) * ldx]));
  }
  if (nc <= 0) return;                                  // uniform over the CTA
  double vals[NV];
#pragma unroll
  for (int c = 0; c < HH_CH; ++c) s_put(vals + c * W, acc[c]);
  double* pch = part + (size_t)ch * HH_GRID_MAX * NV;
  if (hh_cta_partial<NV>(vals, pch, ctr + ch))
    hh_grid_total<NV>(pch, nc * W, reinterpret_cast<double*>(red_w + ch * HH_CH), ctr + ch);
}

// X[:, j+1:pend] -= conj(tau_j) v_j w (the H_j^H update of the rest of the panel; CTA (r, ch) as
// in hh_reflect_kernel), then (chunk 0) the (norm, alpha) partials of column j+1.
template <typename T>
__global__ void __launch_bounds__(HH_THREADS)
    hh_update_kernel(T* X, long long ldx, int n_r, long long voff, int j, int pend, const T* Vp,
                     long long ldvp, int jj, const T* red_w, const T* tau, double* part_n,
                     double* red_n, unsigned* ctr_n) {
  const T ct = s_conj(tau[j]);
  const int ch = blockIdx.y;
  const int nw = pend - j - 1, c0 = j + 1 + ch * HH_CH;
  const int nc = min(HH_CH, nw - ch * HH_CH);
  T w[HH_CH];
#pragma unroll
  for (int c = 0; c < HH_CH; ++c) w[c] = c < nc ? s_mul(ct, red_w[ch * HH_CH + c]) : s_real<T>(0.0);
  const T* vpc = Vp + (long long)jj * ldvp;
  double v3[3] = {0.0, 0.0, 0.0};
  for (int l = blockIdx.x * HH_THREADS + threadIdx.x; l < n_r; l += gridDim.x * HH_THREADS) {
    const long long g = voff + l;
    if (g < j) continue;
    const T v = vpc[l];
#pragma unroll
    for (int c = 0; c < HH_CH; ++c) {
      if (c < nc) {
        T* p = X + (long long)l + (long long)(c0 + c) * ldx;
        const T x = s_sub(*p, s_mul(v, w[c]));
        *p = x;
        if (ch == 0 && c == 0) {
          if (g > j + 1) v3[0] += s_abs2(x);
          else if (g == j + 1) { v3[1] = s_re(x); v3[2] = s_im(x); }
        }
      }
    }
  }
  if (ch == 0 && hh_cta_partial<3>(v3, part_n, ctr_n)) hh_grid_total<3>(part_n, 3, red_n, ctr_n);
}

// After a panel: X[:, j0:pend] <- the LAPACK storage (v_j strictly below the pivot, beta_j on it)
template <typename T>
__global__ void hh_store_panel_kernel(T* X, long long ldx, int n_r, long long voff, int j0,
                                      const T* Vp, long long ldvp, const double* beta) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  const int jj = blockIdx.y;
  if (l >= n_r) return;
  const long long g = voff + l, j = j0 + jj;
  if (g > j) X[(long long)l + j * ldx] = Vp[(long long)l + (long long)jj * ldvp];
  else if (g == j) X[(long long)l + j * ldx] = s_real<T>(beta[j]);
}

// Compact-WY factor of one panel (xLARFT, forward, columnwise) from S = Vp^H Vp (reduced):
//   T[i, i] = tau_i,  T[0:i, i] = T[0:i, 0:i] z,  z = -tau_i S[0:i, i].
// One CTA of HH_NB threads (thread r owns row r); T is HH_NB x HH_NB in global memory (ld
// HH_NB), zero below the diagonal and past nb.
template <typename T>
__global__ void __launch_bounds__(HH_NB) hh_larft_kernel(const T* S, int lds, const T* tau, int j0,
                                                         int nb, T* Tout) {
  __shared__ T z[HH_NB];
  const int r = threadIdx.x;
  for (int c = 0; c < HH_NB; ++c) Tout[r + (long long)c * HH_NB] = s_real<T>(0.0);
  __syncthreads();
  for (int i = 0; i < nb; ++i) {
    const T ti = tau[j0 + i];
    if (r < i) z[r] = s_sub(s_real<T>(0.0), s_mul(ti, S[r + (long long)i * lds]));
    __syncthreads();
    if (r < i) {
      T acc = s_real<T>(0.0);
      for (int m = r; m < i; ++m) acc = s_add(acc, s_mul(Tout[r + (long long)m * HH_NB], z[m]));
      Tout[r + (long long)i * HH_NB] = acc;
    }
    if (r == i) Tout[i + (long long)i * HH_NB] = ti;
    __syncthreads();
  }
}

// split-K partial sums, fixed order: out[i, c] = sum_s part[s * split_ld + i + c * ldp]
template <typename T>
__global__ void hh_splitsum_kernel(const T* part, long long split_ld, int S, int M, int ldp,
                                   T* out, int ldo) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const long long c = blockIdx.y;
  if (i >= M) return;
  T acc = part[i + c * ldp];
  for (int s = 1; s < S; ++s) acc = s_add(acc, part[(long long)s * split_ld + i + c * ldp]);
  out[i + c * ldo] = acc;
}

// Vp[:, jj] = v_{j0+jj} rebuilt from the factored X (zeros above the pivot, 1 at it).
template <typename T>
__global__ void hh_build_vp_kernel(const T* X, long long ldx, int n_r, long long voff, int j0,
                                   int nb, T* Vp, long long ldvp) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  const int jj = blockIdx.y;
  if (l >= n_r) return;
  const long long g = voff + l, j = j0 + jj;
  T v;
  if (jj >= nb || g < j) v = s_real<T>(0.0);
  else if (g == j) v = s_real<T>(1.0);
  else v = X[(long long)l + j * ldx];
  Vp[(long long)l + (long long)jj * ldvp] = v;
}

// Q = [I_n; 0] in virtual rows
template <typename T>
__global__ void hh_init_q_kernel(T* Q, long long ldq, int n_r, long long voff) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  const long long c = blockIdx.y;
  if (l < n_r) Q[(long long)l + c * ldq] = s_real<T>(voff + l == c ? 1.0 : 0.0);
}

// V[:, c] = sign(beta_c) Q[:, c]   (diag(R) made non-negative)
template <typename T>
__global__ void hh_finish_kernel(const T* Q, long long ldq, int n_r, const double* beta, T* V,
                                 long long ldv) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  const long long c = blockIdx.y;
  if (l >= n_r) return;
  const T q = Q[(long long)l + c * ldq];
  V[(long long)l + c * ldv] = beta[c] < 0.0 ? s_sub(s_real<T>(0.0), q) : q;
}

}  // namespace chase
