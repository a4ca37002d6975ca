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
  if constexpr (NV % 32 == 0) {
    // warp reduce-scatter butterfly per group of 32 values (31 shuffles instead of 160): after the
    // step with mask o a lane keeps the partial sums of the values whose index agrees with the
    // lane in bit o; lane l ends with the warp total of value l of the group
#pragma unroll
    for (int base = 0; base < NV; base += 32) {
      double x[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) x[k] = v[base + k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int k = 0; k < o; ++k) {
          const double send = up ? x[k] : x[k + o];
          const double keep = up ? x[k + o] : x[k];
          x[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      wsum[warp][base + lane] = x[0];
    }
  } else {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double x = v[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) wsum[warp][k] = x;
    }
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

// fixed-order sum over the CTA partials (last CTA only); resets the arrival counter.  All
// threads take part: GR groups of threads sum interleaved subsets of the CTA partials (loads of
// a group in flight together), then the GR group sums are added in fixed order.
template <int NV>
__device__ void hh_grid_total(const double* part, int nv, double* out, unsigned* ctr) {
  constexpr int GR = NV >= HH_THREADS ? 1 : (HH_THREADS / NV > 8 ? 8 : HH_THREADS / NV);
  __shared__ double gsum[GR][NV];
  const int k = threadIdx.x % NV, grp = threadIdx.x / NV;
  const int nb = (int)gridDim.x;
  if (grp < GR && k < nv) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int b = grp;
    for (; b + 3 * GR < nb; b += 4 * GR) {
      a0 += __ldcg(part + (size_t)b * NV + k);
      a1 += __ldcg(part + (size_t)(b + GR) * NV + k);
      a2 += __ldcg(part + (size_t)(b + 2 * GR) * NV + k);
      a3 += __ldcg(part + (size_t)(b + 3 * GR) * NV + k);
    }
    for (; b < nb; b += GR) a0 += __ldcg(part + (size_t)b * NV + k);
    gsum[grp][k] = (a0 + a1) + (a2 + a3);
  }
  __syncthreads();
  for (int kk = threadIdx.x; kk < nv; kk += HH_THREADS) {
    double x = 0.0;
#pragma unroll
    for (int g = 0; g < GR; ++g) x += gsum[g][kk];
    out[kk] = x;
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
    T xv[HH_CH];
#pragma unroll
    for (int c = 0; c < HH_CH; ++c)
      if (c < nc) xv[c] = X[(long long)l + (long long)(c0 + c) * ldx];
    const T v = g == j ? s_real<T>(1.0) : s_mul(colj[l], inv);
    if (ch == 0) vpc[l] = v;
#pragma unroll
    for (int c = 0; c < HH_CH; ++c)
      if (c < nc) acc[c] = s_add(acc[c], s_cmul(v, xv[c]));
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
    T* row = X + (long long)l + (long long)c0 * ldx;
    T xv[HH_CH];
#pragma unroll
    for (int c = 0; c < HH_CH; ++c)          // all loads first (the stores below may alias them
      if (c < nc) xv[c] = row[(long long)c * ldx];   // as far as the compiler knows)
#pragma unroll
    for (int c = 0; c < HH_CH; ++c) {
      if (c < nc) {
        const T x = s_sub(xv[c], s_mul(v, w[c]));
        row[(long long)c * ldx] = x;
        if (ch == 0 && c == 0) {
          if (g > j + 1) v3[0] += s_abs2(x);
          else if (g == j + 1) { v3[1] = s_re(x); v3[2] = s_im(x); }
        }
      }
    }
  }
  if (ch == 0 && hh_cta_partial<3>(v3, part_n, ctr_n)) hh_grid_total<3>(part_n, 3, red_n, ctr_n);
}

// ---------------------------------------------------------------------------------------------
// The whole panel [j0, pend) as ONE persistent kernel (column communicator of one member, p == 1):
// the per-column steps of hh_norm / hh_reflect / hh_update with grid-wide barriers instead of
// kernel boundaries (3 per column instead of 2 launches with a last-CTA reduction each).
// Cooperative launch (all CTAs co-resident); CTA b owns the virtual rows
// [b R, (b+1) R), R = ceil(n_r / gridDim.x).  Per column j:
//   (a) every CTA sums the G partials of (||x_{>j}||^2, alpha) in fixed order -> xLARFG
//       reflector (identical in every CTA); v_j into Vp[:, jj]; CTA partials of w = v_j^H X_panel
//   (b) barrier; CTA b totals w for the columns c = b, b + G, ... (fixed order) -> wtot
//   (c) barrier; X_panel -= conj(tau) v_j w on own rows, partials of column j+1's (norm, alpha)
//   (d) barrier
// Deterministic (fixed-order sums), identical to the launch-per-column path up to summation
// order.  Workspace: part (G x (1 + nb) x 2 words ... see hhqr.inc), wtot (nb words), bar (2 u32).
__device__ __forceinline__ void hh_grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned target = gen + 1;
    if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicExch(&bar[1], target);
    } else {
      while (*(volatile unsigned*)&bar[1] != target) __nanosleep(20);
    }
    __threadfence();
  }
  ++gen;
  __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(HH_THREADS)
    hh_panel_kernel(T* X, long long ldx, int n_r, long long voff, int j0, int pend, T* Vp,
                    long long ldvp, T* tau_out, double* beta_out, double* part, T* wtot,
                    unsigned* bar) {
  constexpr int W = s_words<T>();
  constexpr int NWARP = HH_THREADS / 32;
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int R = (n_r + G - 1) / G, r0 = b * R, r1 = min(n_r, r0 + R);
  const int nb = pend - j0;
  // part layout: [0, 3G): (norm, alpha) partials; [3G, 3G + G nb W): w partials (CTA-major)
  double* pn = part;
  double* pw = part + 3 * G;
  __shared__ double red[NWARP][HH_CH * 2];
  __shared__ T sw[HH_NB];
  unsigned gen = *(volatile unsigned*)&bar[1];
  // CTA sum of a per-thread value set (nv <= 2 HH_CH doubles), fixed order.  Within a warp a
  // reduce-scatter butterfly over 32 values (31 shuffles instead of 160): after step o, lane l
  // keeps the partial sums of the values whose index agrees with l in the bits already folded;
  // at the end lane l holds the warp total of value l.  Then the warps in order 0..7.
  auto cta_sum = [&](double* v, int nv, double* dst) {
    for (int base = 0; base < nv; base += 32) {
      double x[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) x[k] = base + k < nv ? v[base + k] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int k = 0; k < o; ++k) {
          // keep x[k] (values with bit o clear) or x[k + o] (bit o set); send the other
          const double send = up ? x[k] : x[k + o];
          const double keep = up ? x[k + o] : x[k];
          x[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      if (base + lane < nv) red[warp][base + lane] = x[0];
    }
    __syncthreads();
    for (int k = tid; k < nv; k += HH_THREADS) {
      double x = 0.0;
#pragma unroll
      for (int w = 0; w < NWARP; ++w) x += red[w][k];
      dst[k] = x;
    }
    __syncthreads();
  };
  // initial (norm, alpha) partials of column j0
  {
    double v3[3] = {0.0, 0.0, 0.0};
    for (int l = r0 + tid; l < r1; l += HH_THREADS) {
      const long long g = voff + l;
      const T x = X[(long long)l + (long long)j0 * ldx];
      if (g > j0) v3[0] += s_abs2(x);
      else if (g == j0) { v3[1] = s_re(x); v3[2] = s_im(x); }
    }
    cta_sum(v3, 3, pn + 3 * b);
  }
  hh_grid_barrier(bar, gen);
  for (int jj = 0; jj < nb; ++jj) {
    const int j = j0 + jj, nw = pend - j - 1;
    // (a) reflector from the fixed-order total of the partials (same in every CTA)
    double tot[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < 3; ++k)
      for (int bb = 0; bb < G; ++bb) tot[k] += __ldcg(pn + 3 * bb + k);
    double beta;
    T tau, inv;
    hh_reflector<T>(tot, &beta, &tau, &inv);
    if (b == 0 && tid == 0) {
      tau_out[j] = tau;
      beta_out[j] = beta;
    }
    // v_j on own rows; w partials in chunks of HH_CH columns
    for (int c0 = 0; c0 < nw; c0 += HH_CH) {
      const int nc = min(HH_CH, nw - c0);
      T acc[HH_CH];
#pragma unroll
      for (int c = 0; c < HH_CH; ++c) acc[c] = s_real<T>(0.0);
      for (int l = r0 + tid; l < r1; l += HH_THREADS) {
        const long long g = voff + l;
        if (g < j) {
          if (c0 == 0) Vp[(long long)l + (long long)jj * ldvp] = s_real<T>(0.0);
          continue;
        }
        const T v = g == j ? s_real<T>(1.0) : s_mul(X[(long long)l + (long long)j * ldx], inv);
        if (c0 == 0) Vp[(long long)l + (long long)jj * ldvp] = v;
#pragma unroll
        for (int c = 0; c < HH_CH; ++c)
          if (c < nc) acc[c] = s_add(acc[c], s_cmul(v, X[(long long)l + (long long)(j + 1 + c0 + c) * ldx]));
      }
      double vals[HH_CH * W];
#pragma unroll
      for (int c = 0; c < HH_CH; ++c) s_put(vals + c * W, acc[c]);
      cta_sum(vals, nc * W, pw + ((size_t)b * HH_NB + c0) * W);
    }
    if (nw <= 0) {   // last column of the panel: v_j only
      for (int l = r0 + tid; l < r1; l += HH_THREADS) {
        const long long g = voff + l;
        const T v = g < j ? s_real<T>(0.0) : (g == j ? s_real<T>(1.0) : s_mul(X[(long long)l + (long long)j * ldx], inv));
        Vp[(long long)l + (long long)jj * ldvp] = v;
      }
      break;
    }
    hh_grid_barrier(bar, gen);
    // (b) w totals, columns c = b, b + G, ... (fixed order over the CTAs)
    for (int c = b + tid * G; c < nw; c += HH_THREADS * G) {
      double x[W];
#pragma unroll
      for (int k = 0; k < W; ++k) x[k] = 0.0;
      for (int bb = 0; bb < G; ++bb)
#pragma unroll
        for (int k = 0; k < W; ++k) x[k] += __ldcg(pw + ((size_t)bb * HH_NB + c) * W + k);
      double* dst = reinterpret_cast<double*>(wtot + c);
#pragma unroll
      for (int k = 0; k < W; ++k) dst[k] = x[k];
    }
    hh_grid_barrier(bar, gen);
    // (c) X_panel -= conj(tau) v w on own rows; (norm, alpha) partials of column j + 1
    for (int c = tid; c < nw; c += HH_THREADS) sw[c] = s_mul(s_conj(tau), __ldcg(wtot + c));
    __syncthreads();
    double v3[3] = {0.0, 0.0, 0.0};
    for (int l = r0 + tid; l < r1; l += HH_THREADS) {
      const long long g = voff + l;
      if (g < j) continue;
      const T v = Vp[(long long)l + (long long)jj * ldvp];
      T* row = X + (long long)l + (long long)(j + 1) * ldx;
      for (int c0 = 0; c0 < nw; c0 += HH_CH) {
        T xv[HH_CH];
#pragma unroll
        for (int c = 0; c < HH_CH; ++c)
          if (c0 + c < nw) xv[c] = row[(long long)(c0 + c) * ldx];
#pragma unroll
        for (int c = 0; c < HH_CH; ++c)
          if (c0 + c < nw) row[(long long)(c0 + c) * ldx] = xv[c] = s_sub(xv[c], s_mul(v, sw[c0 + c]));
        if (c0 == 0) {
          if (g > j + 1) v3[0] += s_abs2(xv[0]);
          else if (g == j + 1) { v3[1] = s_re(xv[0]); v3[2] = s_im(xv[0]); }
        }
      }
    }
    cta_sum(v3, 3, pn + 3 * b);
    hh_grid_barrier(bar, gen);
  }
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
