// qr_kernels.cuh -- the latency-bound pieces of 1D-CholeskyQR (Alg.3; Alg.4 l.5-7,
// P:294-297), templated on double (real symmetric) / double2 (complex Hermitian).  The
// flop-heavy pieces (Gram X^H X, the trailing HERK update of the blocked POTRF, the TRSM
// diagonal-block products and right-looking updates) run on the tensor-core GEMMs.
//
//   potrf_diag_kernel    upper Cholesky of one nb x nb diagonal block and its inverse, in smem
//                        (the block row R[kb, kb+nb:] = R_kk^{-H} G[kb, kb+nb:] is then a GEMM)
//   trtri_diag_kernel    inverses of the 64 x 64 diagonal blocks of R (blocked TRSM)
//   shift_kernel         norm = Re tr(G) (= ||X||_F^2, reading #12); s = 11(mn+n(n+1)) u norm;
//                        G += s I
// A POTRF failure (radicand <= 0 or NaN) writes the 1-based global pivot into *info once;
// every later kernel of the same factorisation sees *info != 0 and returns.
#pragma once
#include "common.cuh"

namespace chase {

constexpr int QR_NB = 64;   // diagonal block size of the blocked POTRF

// scalar ops for T = double (real symmetric) or double2 (complex Hermitian)
__device__ __forceinline__ double2 s_mul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double s_mul(double a, double b) { return a * b; }
__device__ __forceinline__ double2 s_cmul(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double s_cmul(double a, double b) { return a * b; }
__device__ __forceinline__ double2 s_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 s_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double s_add(double a, double b) { return a + b; }
__device__ __forceinline__ double s_sub(double a, double b) { return a - b; }
__device__ __forceinline__ double2 s_div(double2 a, double r) { return make_double2(a.x / r, a.y / r); }
__device__ __forceinline__ double2 s_mulr(double2 a, double r) { return make_double2(a.x * r, a.y * r); }
__device__ __forceinline__ double s_mulr(double a, double r) { return a * r; }
__device__ __forceinline__ double s_div(double a, double r) { return a / r; }
__device__ __forceinline__ double s_re(double2 a) { return a.x; }
__device__ __forceinline__ double s_re(double a) { return a; }
template <typename T> __device__ __forceinline__ T s_real(double r);
template <> __device__ __forceinline__ double2 s_real<double2>(double r) { return make_double2(r, 0.0); }
template <> __device__ __forceinline__ double s_real<double>(double r) { return r; }
__device__ __forceinline__ void s_add_re(double2& a, double v) { a.x += v; }
__device__ __forceinline__ double s_abs2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double s_abs2(double a) { return a * a; }
__device__ __forceinline__ void s_add_re(double& a, double v) { a += v; }

// One CTA of POTRF_DIAG_THREADS.  G column-major (ld), block rows/cols [kb, kb+nb), nb <= 64.
// On exit the upper triangle of the block holds R_kk (real positive diagonal) and, when Rinv is
// not null, Rinv[0:nb, 0:nb] (ld 64) holds R_kk^{-1} (upper, zeros below), from which the block
// row R[kb, kb+nb:] = R_kk^{-H} G[kb, kb+nb:] is one tensor-core GEMM (chase.cu, cholqr_pass).
//  * factorisation: right-looking, column j at a time; the trailing update of the upper triangle
//    is spread evenly over all threads through a table of the (a, b) pairs, a <= b, ordered by a
//    descending, so step j updates exactly the first (nb-1-j)(nb-j)/2 entries;
//  * inverse: recursive doubling in smem -- X_ii = 1/R_ii, then for w = 1, 2, .., 32 every
//    pair of inverted w-blocks becomes a 2w-block, X12 = -X11 (R12 X22).
// A non-positive (or NaN) pivot writes the 1-based global pivot into *info and returns.
constexpr int POTRF_DIAG_THREADS = 256;
template <typename T>
constexpr int diag_smem() { return 3 * QR_NB * (QR_NB + 1) * (int)sizeof(T) + QR_NB * (QR_NB + 1) / 2 * 2; }
template <typename T>
__global__ void __launch_bounds__(POTRF_DIAG_THREADS)
    potrf_diag_kernel(T* G, long long ld, int kb, int nb, int* info, T* Rinv) {
  extern __shared__ __align__(16) unsigned char qr_dyn[];
  constexpr int LD = QR_NB + 1;
  T (*S)[LD] = reinterpret_cast<T (*)[LD]>(qr_dyn);                              // R
  T (*X)[LD] = reinterpret_cast<T (*)[LD]>(qr_dyn + QR_NB * LD * sizeof(T));     // R^{-1}
  T (*W)[LD] = reinterpret_cast<T (*)[LD]>(qr_dyn + 2 * QR_NB * LD * sizeof(T)); // temp
  unsigned short* tab = reinterpret_cast<unsigned short*>(qr_dyn + 3 * QR_NB * LD * sizeof(T));
  if (*info != 0) return;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < nb * nb; idx += POTRF_DIAG_THREADS) {   // coalesced: rows fastest
    const int a = idx % nb, c = idx / nb;
    S[a][c] = G[(long long)(kb + a) + (long long)(kb + c) * ld];
  }
  // pair table: entry e <-> (a, b), a <= b < nb, a descending: pairs with a = nb-1-q start at
  // q(q+1)/2; thread-parallel fill
  const int npairs = nb * (nb + 1) / 2;
  for (int e = tid; e < npairs; e += POTRF_DIAG_THREADS) {
    int q = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);                  // largest q, q(q+1)/2 <= e
    while ((q + 1) * (q + 2) / 2 <= e) ++q;
    while (q * (q + 1) / 2 > e) --q;
    const int a = nb - 1 - q, b = a + (e - q * (q + 1) / 2);
    tab[e] = (unsigned short)((a << 8) | b);
  }
  __syncthreads();
  // one barrier per column: row j is used unscaled (conj(R_ja) R_jb = conj(S_ja) S_jb / d_j) and
  // scaled by 1/sqrt(d_j) only after the loop -- rows <= j are never written after step j
  for (int j = 0; j < nb; ++j) {
    const double d = s_re(S[j][j]);
    if (!(d > 0.0)) {                       // uniform: every thread reads the same d
      if (tid == 0) atomicCAS(info, 0, kb + j + 1);
      return;
    }
    const double dinv = 1.0 / d;
    // S[a][b] -= conj(S[j][a]) S[j][b] / d for j < a <= b < nb: the first cnt table entries
    const int cnt = (nb - 1 - j) * (nb - j) / 2;
    for (int e = tid; e < cnt; e += POTRF_DIAG_THREADS) {
      const int a = tab[e] >> 8, b = tab[e] & 255;
      S[a][b] = s_sub(S[a][b], s_mulr(s_cmul(S[j][a], S[j][b]), dinv));
    }
    __syncthreads();
  }
  // R[j][j] = sqrt(d_j), R[j][b] = S[j][b] / sqrt(d_j) (b > j)
  for (int idx = tid; idx < nb * nb; idx += POTRF_DIAG_THREADS) {
    const int a = idx % nb, c = idx / nb;
    if (a < c) S[a][c] = s_mulr(S[a][c], 1.0 / sqrt(s_re(S[a][a])));
  }
  __syncthreads();
  for (int a = tid; a < nb; a += POTRF_DIAG_THREADS) S[a][a] = s_real<T>(sqrt(s_re(S[a][a])));
  __syncthreads();
  for (int idx = tid; idx < nb * nb; idx += POTRF_DIAG_THREADS) {   // coalesced store (upper)
    const int a = idx % nb, c = idx / nb;
    if (a <= c) G[(long long)(kb + a) + (long long)(kb + c) * ld] = S[a][c];
  }
  if (Rinv == nullptr) return;
  // inverse by recursive doubling
  for (int idx = tid; idx < QR_NB * QR_NB; idx += POTRF_DIAG_THREADS) {
    const int a = idx % QR_NB, c = idx / QR_NB;
    X[a][c] = (a == c && a < nb) ? s_real<T>(1.0 / s_re(S[a][a])) : s_real<T>(0.0);
  }
  __syncthreads();
  for (int w = 1; w < nb; w *= 2) {
    // W[i0:j0, j0:j0+w2] = R12 X22 for every pair (i0 = 2 w p, j0 = i0 + w, w2 = min(w, nb - j0))
    const int npair = (nb - w + 2 * w - 1) / (2 * w);
    for (int e = tid; e < npair * w * w; e += POTRF_DIAG_THREADS) {
      const int p = e / (w * w), r = (e % (w * w)) % w, c = (e % (w * w)) / w;
      const int i0 = 2 * w * p, j0 = i0 + w;
      if (j0 + c >= nb) continue;
      T acc = s_real<T>(0.0);
      for (int k = 0; k <= c; ++k) acc = s_add(acc, s_mul(S[i0 + r][j0 + k], X[j0 + k][j0 + c]));
      W[i0 + r][j0 + c] = acc;
    }
    __syncthreads();
    // X12 = -X11 W (X11 upper: k from r)
    for (int e = tid; e < npair * w * w; e += POTRF_DIAG_THREADS) {
      const int p = e / (w * w), r = (e % (w * w)) % w, c = (e % (w * w)) / w;
      const int i0 = 2 * w * p, j0 = i0 + w;
      if (j0 + c >= nb) continue;
      T acc = s_real<T>(0.0);
      for (int k = r; k < w; ++k) acc = s_add(acc, s_mul(X[i0 + r][i0 + k], W[i0 + k][j0 + c]));
      X[i0 + r][j0 + c] = s_sub(s_real<T>(0.0), acc);
    }
    __syncthreads();
  }
  for (int idx = tid; idx < QR_NB * QR_NB; idx += POTRF_DIAG_THREADS) {
    const int a = idx % QR_NB, c = idx / QR_NB;
    Rinv[(long long)a + (long long)c * QR_NB] = (a < nb && c < nb && a <= c) ? X[a][c] : s_real<T>(0.0);
  }
}

// Inverses of the diagonal blocks of the upper-triangular R: CTA b inverts
// R[kb:kb+nb, kb:kb+nb], kb = 64 b, into Rinv[0:64, kb:kb+64] (full == 0: compact, ld 64, zeros
// below the diagonal and in the padding of a short last block) or into the diagonal block
// Rinv[kb:kb+nb, kb:kb+nb] of an n x n matrix with leading dimension ldr (full == 1, the seed of
// the recursive-doubling inverse of R; nothing outside the block is written).
// Thread j solves R_kk x = e_j by back substitution:
//   x_j = 1 / R_jj,  x_i = -(sum_{l=i+1..j} R_il x_l) / R_ii   (i = j-1 .. 0).
constexpr int TRTRI_NB = 64;
template <typename T>
constexpr int trtri_smem() { return 2 * TRTRI_NB * TRTRI_NB * (int)sizeof(T); }
template <typename T>
__global__ void __launch_bounds__(TRTRI_NB)
    trtri_diag_kernel(const T* G, long long ld, int n, T* Rinv, long long ldr = TRTRI_NB, int full = 0) {
  extern __shared__ __align__(16) unsigned char qr_dyn[];
  T (*R)[TRTRI_NB] = reinterpret_cast<T (*)[TRTRI_NB]>(qr_dyn);                 // R[i][l]
  T (*X)[TRTRI_NB] = reinterpret_cast<T (*)[TRTRI_NB]>(qr_dyn + TRTRI_NB * TRTRI_NB * sizeof(T));
  const int kb = blockIdx.x * TRTRI_NB;
  const int nb = min(TRTRI_NB, n - kb);
  const int j = threadIdx.x;
  for (int idx = j; idx < TRTRI_NB * TRTRI_NB; idx += TRTRI_NB) {
    const int a = idx % TRTRI_NB, b = idx / TRTRI_NB;
    R[a][b] = (a < nb && b < nb && a <= b) ? G[(long long)(kb + a) + (long long)(kb + b) * ld]
                                           : s_real<T>(0.0);
  }
  __syncthreads();
  for (int i = 0; i < TRTRI_NB; ++i) X[i][j] = s_real<T>(0.0);
  if (j < nb) {
    X[j][j] = s_real<T>(1.0 / s_re(R[j][j]));
    for (int i = j - 1; i >= 0; --i) {
      T a0 = s_real<T>(0.0), a1 = s_real<T>(0.0);
      int l = i + 1;
      for (; l + 1 <= j; l += 2) {
        a0 = s_sub(a0, s_mul(R[i][l], X[l][j]));
        a1 = s_sub(a1, s_mul(R[i][l + 1], X[l + 1][j]));
      }
      if (l <= j) a0 = s_sub(a0, s_mul(R[i][l], X[l][j]));
      X[i][j] = s_div(s_add(a0, a1), s_re(R[i][i]));
    }
  }
  if (full) {
    if (j < nb)
      for (int i = 0; i < nb; ++i) Rinv[(long long)(kb + i) + (long long)(kb + j) * ldr] = X[i][j];
  } else {
    for (int i = 0; i < TRTRI_NB; ++i) Rinv[(long long)i + (long long)(kb + j) * ldr] = X[i][j];
  }
}

// Residual norms, Alg.2 l.26 "nrm <- SquaredNorm(B)": nrm[c] = sum_r |B[r, c]|^2 over the local
// rows of the B-layout block.  One CTA per column, fixed-order tree reduction (deterministic).
template <typename T>
__global__ void colnorm2_kernel(const T* B, long long ld, int rows, double* nrm) {
  __shared__ double part[256];
  const int tid = threadIdx.x;
  const long long col = blockIdx.x;
  double acc = 0.0;
  for (int r = tid; r < rows; r += 256) {
    const T v = B[(long long)r + col * ld];
    acc += s_abs2(v);
  }
  part[tid] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (tid < w) part[tid] += part[tid + w];
    __syncthreads();
  }
  if (tid == 0) nrm[col] = part[0];
}

// Block-cyclic B2 redistribution (Alg.2 l.23 on a cyclic grid): gather local rows idx[0..cnt)
// of V into a dense cnt x ncols stage (ld cnt), and scatter a stage into rows idx of B2.
template <typename T>
__global__ void gather_rows_kernel(const T* V, long long ldv, const int* idx, int cnt, T* stage) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const long long col = blockIdx.y;
  if (i < cnt) stage[(long long)i + col * cnt] = V[(long long)idx[i] + col * ldv];
}
template <typename T>
__global__ void scatter_rows_kernel(const T* stage, const int* idx, int cnt, T* B2, long long ldb) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const long long col = blockIdx.y;
  if (i < cnt) B2[(long long)idx[i] + col * ldb] = stage[(long long)i + col * cnt];
}

// Alg.2 l.28 "resd <- sqrt(nrm)" on the reduced squared norms.
__global__ void sqrt_kernel(double* v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = sqrt(v[i]);
}

// Alg.4 l.5-7 on the reduced Gram matrix: norm = sum_j Re G[j][j]; s = 11 (m n + n (n+1)) u norm;
// G[j][j] += s.  One CTA of 256 threads, fixed-order reduction (deterministic).
template <typename T>
__global__ void shift_kernel(T* G, long long ld, int n, long long m_global, double* s_out) {
  __shared__ double part[256];
  const int tid = threadIdx.x;
  double acc = 0.0;
  for (int j = tid; j < n; j += 256) acc += s_re(G[(long long)j + (long long)j * ld]);
  part[tid] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (tid < w) part[tid] += part[tid + w];
    __syncthreads();
  }
  const double norm = part[0];
  const double u = 1.1102230246251565e-16;   // 2^-53
  const double s = 11.0 * (double)(m_global * (long long)n + (long long)n * (n + 1)) * u * norm;
  for (int j = tid; j < n; j += 256) s_add_re(G[(long long)j + (long long)j * ld], s);
  if (tid == 0 && s_out != nullptr) *s_out = s;
}

}  // namespace chase
