// chase_oracle.cpp -- CPU ORACLE (TEST INFRASTRUCTURE ONLY) for the ChASE hot path of
// arXiv 2309.15595: the plain, slow, triple-loop Chebyshev filter and CholeskyQR family the
// BASELINE north star asks for ("a plain, slow CPU filter and CholeskyQR with triple loops,
// sharing no code with the GPU path").  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it; the product path (libchase.so) never does.
//
// C++17, std::complex<double>, OpenMP over output rows, built -O2 -fno-fast-math
// -ffp-contract=off (no reassociation, no FMA contraction) -fcx-limited-range (complex products
// by the textbook formula (ac - bd) + i(ad + bc), without the C99 Annex G NaN recovery).
// Shares no code, header or constant with csrc/: every
// formula is written out here from the paper, in its notation (P:NNN = PAPER.md line,
// S:NNN = SPEC.md line, readings #k = DESIGN.md §3).  Pinned by tests/test_oracle_cpp.py against
// closed forms (Chebyshev values on diagonal / Q diag(lambda) Q^H matrices), the golden hand
// cases of tests/golden/, LAPACK and QR invariants -- the same pins as the numpy oracle.
//
// Matrices are column-major; complex data is interleaved (re, im) doubles.  Element (r, c) of an
// m x n matrix X with leading dimension ld is X[r + c * ld].
#include <cmath>
#include <complex>
#include <cstdint>
#include <vector>

typedef std::complex<double> zc;

namespace {

// Eq.(1) scalars with the S:362 damping (reading #1):
//   sigma_1 = e / (mu_1 - c);  alpha_1 = sigma_1 / e, beta_1 = 0;
//   sigma_s = 1 / (2 / sigma_1 - sigma_{s-1}); alpha_s = 2 sigma_s / e; beta_s = -sigma_{s-1} sigma_s
void scalars(double c, double e, double mu_1, int D, std::vector<double>& alpha, std::vector<double>& beta) {
  alpha.assign(D, 0.0);
  beta.assign(D, 0.0);
  const double sigma_1 = e / (mu_1 - c);
  double sigma = sigma_1;
  alpha[0] = sigma_1 / e;
  beta[0] = 0.0;
  for (int s = 2; s <= D; ++s) {
    const double prev = sigma;
    sigma = 1.0 / (2.0 / sigma_1 - prev);
    alpha[s - 1] = 2.0 * sigma / e;
    beta[s - 1] = -prev * sigma;
  }
}

// The filter for element type T (double or complex<double>), global N x N A, N x n V.
//   step s, active column j (d_j >= s):
//     W_new[r, j] = alpha_s (sum_t A[r, t] W[t, j] - c W[r, j]) + beta_s W_old[r, j]
// Column j's result is W after step d_j (reading #3).  Triple loop: rows (OpenMP) x active
// columns x t; A is read column by column (t outer inside a row block) so each pass streams A.
template <typename T>
void filter_impl(int64_t N, int64_t n, const T* A, int64_t lda, T* V, int64_t ldv, const int32_t* deg,
                 double c, double e, double mu_1) {
  int D = 0;
  for (int64_t j = 0; j < n; ++j) D = deg[j] > D ? deg[j] : D;
  std::vector<double> alpha, beta;
  scalars(c, e, mu_1, D, alpha, beta);
  std::vector<T> Wold((size_t)N * n), W((size_t)N * n), Wnew((size_t)N * n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t r = 0; r < N; ++r) W[r + j * N] = V[r + j * ldv];       // W = V_0
  constexpr int64_t RB = 64;                                               // rows per block
  for (int s = 1; s <= D; ++s) {
    int64_t j0 = 0;
    while (j0 < n && deg[j0] < s) ++j0;                                    // active suffix
    const double a = alpha[s - 1], b = beta[s - 1];
#pragma omp parallel for schedule(static)
    for (int64_t r0 = 0; r0 < N; r0 += RB) {
      const int64_t r1 = r0 + RB < N ? r0 + RB : N;
      std::vector<T> acc((size_t)(r1 - r0) * (n - j0), T(0));
      for (int64_t t = 0; t < N; ++t)
        for (int64_t j = j0; j < n; ++j) {
          const T w = W[t + j * N];
          T* ac = &acc[(size_t)(j - j0) * (r1 - r0)];
          for (int64_t r = r0; r < r1; ++r) ac[r - r0] += A[r + t * lda] * w;
        }
      for (int64_t j = j0; j < n; ++j)
        for (int64_t r = r0; r < r1; ++r) {
          const T av = acc[(size_t)(j - j0) * (r1 - r0) + (r - r0)];
          T v = a * (av - c * W[r + j * N]);
          if (s > 1) v += b * Wold[r + j * N];
          Wnew[r + j * N] = v;
        }
    }
    for (int64_t j = j0; j < n; ++j)
      for (int64_t r = 0; r < N; ++r) {
        Wold[r + j * N] = W[r + j * N];
        W[r + j * N] = Wnew[r + j * N];
      }
    for (int64_t j = j0; j < n; ++j)
      if (deg[j] == s)
        for (int64_t r = 0; r < N; ++r) V[r + j * ldv] = W[r + j * N];   // column j retires
  }
}

inline double conj_(double x) { return x; }
inline zc conj_(const zc& x) { return std::conj(x); }
inline double re_(double x) { return x; }
inline double re_(const zc& x) { return x.real(); }
inline double abs2_(double x) { return x * x; }
inline double abs2_(const zc& x) { return x.real() * x.real() + x.imag() * x.imag(); }

// Alg.3 l.3: G[a, b] = sum_r conj(X[r, a]) X[r, b]  (upper triangle a <= b, mirrored)
template <typename T>
void gram_impl(int64_t m, int64_t n, const T* X, int64_t ldx, T* G) {
#pragma omp parallel for schedule(dynamic)
  for (int64_t b = 0; b < n; ++b)
    for (int64_t a = 0; a <= b; ++a) {
      T s(0);
      for (int64_t r = 0; r < m; ++r) s += conj_(X[r + a * ldx]) * X[r + b * ldx];
      G[a + b * n] = s;
      G[b + a * n] = conj_(s);
    }
}

// Alg.3 l.5: upper Cholesky G = R^H R, row by row:
//   R[j, j] = sqrt(G[j, j] - sum_{k<j} |R[k, j]|^2)   (fail: info = j + 1 if not > 0 or NaN)
//   R[j, l] = (G[j, l] - sum_{k<j} conj(R[k, j]) R[k, l]) / R[j, j],  l > j
template <typename T>
int potrf_impl(int64_t n, const T* G, T* R) {
  for (int64_t i = 0; i < n * n; ++i) R[i] = T(0);
  for (int64_t j = 0; j < n; ++j) {
    double rad = re_(G[j + j * n]);
    for (int64_t k = 0; k < j; ++k) rad -= abs2_(R[k + j * n]);
    if (!(rad > 0.0)) return (int)(j + 1);
    const double rjj = std::sqrt(rad);
    R[j + j * n] = T(rjj);
#pragma omp parallel for schedule(static)
    for (int64_t l = j + 1; l < n; ++l) {
      T s = G[j + l * n];
      for (int64_t k = 0; k < j; ++k) s -= conj_(R[k + j * n]) * R[k + l * n];
      R[j + l * n] = s / rjj;
    }
  }
  return 0;
}

// Alg.3 l.6: X <- X R^{-1} by rows: y_l = (x_l - sum_{k<l} y_k R[k, l]) / R[l, l]
template <typename T>
void trsm_impl(int64_t m, int64_t n, T* X, int64_t ldx, const T* R) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < m; ++r)
    for (int64_t l = 0; l < n; ++l) {
      T s = X[r + l * ldx];
      for (int64_t k = 0; k < l; ++k) s -= X[r + k * ldx] * R[k + l * n];
      X[r + l * ldx] = s / re_(R[l + l * n]);
    }
}

// Alg.4 l.5-6: norm = ||X||_F^2 = sum |x|^2; s = 11 (m n + n (n + 1)) u norm,
// u = 2^-53 (readings #10-#12)
template <typename T>
double shift_impl(int64_t m, int64_t n, const T* X, int64_t ldx) {
  double norm = 0.0;
  for (int64_t b = 0; b < n; ++b)
    for (int64_t r = 0; r < m; ++r) norm += abs2_(X[r + b * ldx]);
  const double u = std::ldexp(1.0, -53);
  return 11.0 * (double)(m * n + n * (n + 1)) * u * norm;
}

// one Alg.3 pass, optionally shifted (Alg.4 l.5-7): 0 on success, else the failing pivot
template <typename T>
int pass_impl(int64_t m, int64_t n, T* X, int64_t ldx, bool shifted, double* s_out) {
  std::vector<T> G((size_t)n * n), R((size_t)n * n);
  gram_impl(m, n, X, ldx, G.data());
  if (shifted) {
    const double s = shift_impl(m, n, X, ldx);
    for (int64_t j = 0; j < n; ++j) G[j + j * n] += s;
    if (s_out) *s_out = s;
  }
  const int info = potrf_impl(n, G.data(), R.data());
  if (info) return info;
  trsm_impl(m, n, X, ldx, R.data());
  return 0;
}

// Alg.4 without the HHQR fallback: est > 1e8 -> one shifted pass + CholeskyQR2;
// est < 20 -> CholeskyQR; else CholeskyQR2 (ties -> CholeskyQR2, reading #9); a failing first
// POTRF of CholeskyQR/CholeskyQR2 escalates to the shifted path (reading #14).  Returns
// 0 (done), or the 1-based pivot of a failure the caller must hand to HHQR (reading #33).
template <typename T>
int caqr_impl(int64_t m, int64_t n, T* X, int64_t ldx, double est, int32_t* variant, int32_t* passes,
              double* shift) {
  int v = est > 1e8 ? 3 : (est < 20.0 ? 1 : 2);
  *passes = 0;
  *shift = 0.0;
  if (v != 3) {
    const int rounds = v == 1 ? 1 : 2;
    for (int i = 0; i < rounds; ++i) {
      const int info = pass_impl(m, n, X, ldx, false, nullptr);
      if (info) {
        if (*passes > 0) {
          *variant = 4;
          return info;
        }
        v = 3;
        break;
      }
      ++*passes;
    }
    if (v != 3) {
      *variant = v;
      return 0;
    }
  }
  *variant = 3;
  int info = pass_impl(m, n, X, ldx, true, shift);
  if (info) {
    *variant = 4;
    return info;
  }
  ++*passes;
  for (int i = 0; i < 2; ++i) {
    info = pass_impl(m, n, X, ldx, false, nullptr);
    if (info) {
      *variant = 4;
      return info;
    }
    ++*passes;
  }
  return 0;
}

}  // namespace

extern "C" {

// The Chebyshev filter (Eq.(1); Alg.1 l.4) in place on V; cplx != 0: interleaved
// complex.  Degrees even, >= 2, non-decreasing (checked by the Python wrapper).
void oracle_cpp_filter(int64_t N, int64_t n, int32_t cplx, const double* A, int64_t lda, double* V,
                       int64_t ldv, const int32_t* degrees, double c, double e, double mu_1) {
  if (cplx)
    filter_impl<zc>(N, n, reinterpret_cast<const zc*>(A), lda, reinterpret_cast<zc*>(V), ldv, degrees, c,
                    e, mu_1);
  else
    filter_impl<double>(N, n, A, lda, V, ldv, degrees, c, e, mu_1);
}

void oracle_cpp_gram(int64_t m, int64_t n, int32_t cplx, const double* X, int64_t ldx, double* G) {
  if (cplx)
    gram_impl<zc>(m, n, reinterpret_cast<const zc*>(X), ldx, reinterpret_cast<zc*>(G));
  else
    gram_impl<double>(m, n, X, ldx, G);
}

int32_t oracle_cpp_potrf(int64_t n, int32_t cplx, const double* G, double* R) {
  return cplx ? potrf_impl<zc>(n, reinterpret_cast<const zc*>(G), reinterpret_cast<zc*>(R))
              : potrf_impl<double>(n, G, R);
}

void oracle_cpp_trsm(int64_t m, int64_t n, int32_t cplx, double* X, int64_t ldx, const double* R) {
  if (cplx)
    trsm_impl<zc>(m, n, reinterpret_cast<zc*>(X), ldx, reinterpret_cast<const zc*>(R));
  else
    trsm_impl<double>(m, n, X, ldx, R);
}

double oracle_cpp_shift(int64_t m, int64_t n, int32_t cplx, const double* X, int64_t ldx) {
  return cplx ? shift_impl<zc>(m, n, reinterpret_cast<const zc*>(X), ldx) : shift_impl<double>(m, n, X, ldx);
}

int32_t oracle_cpp_caqr(int64_t m, int64_t n, int32_t cplx, double* X, int64_t ldx, double est,
                        int32_t* variant, int32_t* passes, double* shift) {
  return cplx ? caqr_impl<zc>(m, n, reinterpret_cast<zc*>(X), ldx, est, variant, passes, shift)
              : caqr_impl<double>(m, n, X, ldx, est, variant, passes, shift);
}

}  // extern "C"
