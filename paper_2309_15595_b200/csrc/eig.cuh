// eig.cuh -- Hermitian eigensolver for the Rayleigh-Ritz quotient (Alg.2 l.20 "HE(SY)EVD(A)",
// P:191): a parallel block two-sided Jacobi method, fully on the GPU.
//
// The n x n quotient (padded to n_p, a multiple of 64) is split into 32-column blocks.  A
// circle-method tournament pairs the blocks; the pairs of a round are made physically adjacent
// (a block permutation of rows/columns between rounds), so pair i owns columns [64 i, 64 i + 64).
// Per round:
//   jacobi_pair_kernel   one CTA per pair: cyclic scalar Jacobi on the 64 x 64 diagonal block in
//                        shared memory (no sorting, so U stays close to the identity) -> U_i
//   GEMM (diag_k = 1)    A[:, pair] <- A[:, pair] U_i,  Y[:, pair] <- Y[:, pair] U_i
//   GEMM (diag_k = 2)    A[pair, :] <- U_i^H A[pair, :]        (tensor cores, U_bd block diagonal)
//   jacobi_perm_kernel   next round's block layout
// until off(A) <= 1e-14 ||A||_F; eigenvalues = diag(A), eigenvectors = columns of Y.  Rotation of
// the 2 x 2 Hermitian [[a_pp, a_pq], [conj(a_pq), a_qq]], a_pq = |a_pq| e:
//   tau = (a_qq - a_pp) / (2 |a_pq|), t = sign(tau) / (|tau| + sqrt(1 + tau^2)), c = 1/sqrt(1+t^2),
//   s = t c;  columns: p' = c p - s conj(e) q,  q' = s e p + c q;  rows: p' = c p - s e q,
//   q' = s conj(e) p + c q.
// Deterministic (fixed orders everywhere), so every rank produces identical bits.
#pragma once
#include "common.cuh"

namespace chase {

constexpr int JAC_PW = 64;                 // pair width = two 32-column blocks = one GEMM n-tile
constexpr int JAC_THREADS = 256;
constexpr int JAC_LD = JAC_PW + 1;
constexpr int JAC_SMEM = 2 * JAC_PW * JAC_LD * 16 + 3 * 32 * 16;

__device__ __forceinline__ void jac_pair_of(int r, int i, int& a, int& b) {
  // circle method for 64 players, round r in [0, 63), game i in [0, 32)
  if (i == 0) {
    a = 63;
    b = r;
  } else {
    a = (r + i) % 63;
    b = (r - i + 63) % 63;
  }
  if (a > b) {
    const int t = a;
    a = b;
    b = t;
  }
}

// One CTA per pair: diagonalise the 64 x 64 block S = A[64 i:, 64 i:] by cyclic Jacobi sweeps,
// write the accumulated unitary into the diagonal block of U_bd.
__global__ void __launch_bounds__(JAC_THREADS)
    jacobi_pair_kernel(const double2* A, long long lda, double2* Ubd, long long ldu, int max_sweeps) {
  extern __shared__ __align__(16) unsigned char jac_smem[];
  double2 (*S)[JAC_LD] = reinterpret_cast<double2 (*)[JAC_LD]>(jac_smem);
  double2 (*U)[JAC_LD] = reinterpret_cast<double2 (*)[JAC_LD]>(jac_smem + JAC_PW * JAC_LD * 16);
  double* rc = reinterpret_cast<double*>(jac_smem + 2 * JAC_PW * JAC_LD * 16);   // c[32]
  double* rs = rc + 32;                                                          // s[32]
  double2* re = reinterpret_cast<double2*>(rs + 32);                             // e[32]
  __shared__ double s_off, s_tot;
  __shared__ int s_rot;
  const int base = blockIdx.x * JAC_PW;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < JAC_PW * JAC_PW; idx += JAC_THREADS) {
    const int r = idx % JAC_PW, c = idx / JAC_PW;
    S[r][c] = A[(long long)(base + r) + (long long)(base + c) * lda];
    U[r][c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int round = 0; round < 63; ++round) {
      if (tid < 32) {
        int p, q;
        jac_pair_of(round, tid, p, q);
        const double app = S[p][p].x, aqq = S[q][q].x;
        const double2 apq = S[p][q];
        const double a = sqrt(apq.x * apq.x + apq.y * apq.y);
        double c = 1.0, s = 0.0;
        double2 e = make_double2(1.0, 0.0);
        if (a > 1e-18 * sqrt(fabs(app * aqq)) && a > 1e-300) {
          e = make_double2(apq.x / a, apq.y / a);
          const double tau = (aqq - app) / (2.0 * a);
          const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          c = 1.0 / sqrt(1.0 + t * t);
          s = t * c;
          s_rot = 1;
        }
        rc[tid] = c;
        rs[tid] = s;
        re[tid] = e;
      }
      __syncthreads();
      // columns of S and U: p' = c p - s conj(e) q,  q' = s e p + c q
      for (int task = tid; task < 32 * JAC_PW; task += JAC_THREADS) {
        const int i = task / JAC_PW, k = task % JAC_PW;
        int p, q;
        jac_pair_of(round, i, p, q);
        const double c = rc[i], s = rs[i];
        const double2 e = re[i];
        const double2 sp = S[k][p], sq = S[k][q];
        // conj(e) q = (e.x q.x + e.y q.y, e.x q.y - e.y q.x); e p = (e.x p.x - e.y p.y, e.x p.y + e.y p.x)
        S[k][p] = make_double2(c * sp.x - s * (e.x * sq.x + e.y * sq.y), c * sp.y - s * (e.x * sq.y - e.y * sq.x));
        S[k][q] = make_double2(s * (e.x * sp.x - e.y * sp.y) + c * sq.x, s * (e.x * sp.y + e.y * sp.x) + c * sq.y);
        const double2 up = U[k][p], uq = U[k][q];
        U[k][p] = make_double2(c * up.x - s * (e.x * uq.x + e.y * uq.y), c * up.y - s * (e.x * uq.y - e.y * uq.x));
        U[k][q] = make_double2(s * (e.x * up.x - e.y * up.y) + c * uq.x, s * (e.x * up.y + e.y * up.x) + c * uq.y);
      }
      __syncthreads();
      // rows of S: p' = c p - s e q,  q' = s conj(e) p + c q
      for (int task = tid; task < 32 * JAC_PW; task += JAC_THREADS) {
        const int i = task / JAC_PW, k = task % JAC_PW;
        int p, q;
        jac_pair_of(round, i, p, q);
        const double c = rc[i], s = rs[i];
        const double2 e = re[i];
        const double2 sp = S[p][k], sq = S[q][k];
        S[p][k] = make_double2(c * sp.x - s * (e.x * sq.x - e.y * sq.y), c * sp.y - s * (e.x * sq.y + e.y * sq.x));
        S[q][k] = make_double2(s * (e.x * sp.x + e.y * sp.y) + c * sq.x, s * (e.x * sp.y - e.y * sp.x) + c * sq.y);
      }
      __syncthreads();
    }
    // stop when this sweep rotated nothing or the block is diagonal to roundoff (parallel,
    // fixed-order reduction)
    {
      double off = 0.0, tot = 0.0;
      for (int idx = tid; idx < JAC_PW * JAC_PW; idx += JAC_THREADS) {
        const int r = idx % JAC_PW, c = idx / JAC_PW;
        const double v = S[r][c].x * S[r][c].x + S[r][c].y * S[r][c].y;
        tot += v;
        if (r != c) off += v;
      }
      for (int o = 16; o > 0; o >>= 1) {
        off += __shfl_xor_sync(0xffffffffu, off, o);
        tot += __shfl_xor_sync(0xffffffffu, tot, o);
      }
      __shared__ double w_off[JAC_THREADS / 32], w_tot[JAC_THREADS / 32];
      if ((tid & 31) == 0) {
        w_off[tid >> 5] = off;
        w_tot[tid >> 5] = tot;
      }
      __syncthreads();
      if (tid == 0) {
        double o2 = 0.0, t2 = 0.0;
        for (int w = 0; w < JAC_THREADS / 32; ++w) {
          o2 += w_off[w];
          t2 += w_tot[w];
        }
        s_off = o2;
        s_tot = t2;
      }
    }
    __syncthreads();
    if (!s_rot || s_off <= 1e-32 * s_tot) break;
    __syncthreads();
  }
  for (int idx = tid; idx < JAC_PW * JAC_PW; idx += JAC_THREADS) {
    const int r = idx % JAC_PW, c = idx / JAC_PW;
    Ubd[(long long)(base + r) + (long long)(base + c) * ldu] = U[r][c];
  }
}

// Block permutation between rounds: new position blocks take old position src[pb] (32-wide).
//   A_new[i][j] = A_old[pi(i)][pi(j)],  Y_new[i][j] = Y_old[i][pi(j)]
__global__ void jacobi_perm_kernel(const double2* Aold, double2* Anew, const double2* Yold,
                                   double2* Ynew, long long ld, int np, const int* src) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)np * np) return;
  const int i = (int)(e % np), j = (int)(e / np);
  const int pi = src[i >> 5] * 32 + (i & 31), pj = src[j >> 5] * 32 + (j & 31);
  Anew[(long long)i + (long long)j * ld] = Aold[(long long)pi + (long long)pj * ld];
  Ynew[(long long)i + (long long)j * ld] = Yold[(long long)i + (long long)pj * ld];
}

// Hermitian part of the n x n quotient and padding to np: A <- (A + A^H)/2 on [0, n)^2, zero
// coupling to the padded indices, padded diagonal = pad (sorts after every eigenvalue).
// Y <- identity, U_bd <- 0.
__global__ void jacobi_init_kernel(double2* A, double2* Y, double2* Ubd, long long ld, int n,
                                   int np, double pad) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)np * np) return;
  const int i = (int)(e % np), j = (int)(e / np);
  Y[e % np + (long long)j * ld] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  Ubd[(long long)i + (long long)j * ld] = make_double2(0.0, 0.0);
  if (i > j) return;                              // (i, j) and (j, i) handled by i <= j
  double2* aij = A + (long long)i + (long long)j * ld;
  double2* aji = A + (long long)j + (long long)i * ld;
  if (i < n && j < n) {
    if (i == j) {
      *aij = make_double2(aij->x, 0.0);
    } else {
      const double2 x = *aij, y = *aji;
      const double2 hh = make_double2(0.5 * (x.x + y.x), 0.5 * (x.y - y.y));
      *aij = hh;
      *aji = make_double2(hh.x, -hh.y);
    }
  } else {
    *aij = make_double2(i == j ? pad : 0.0, 0.0);
    *aji = make_double2(i == j ? pad : 0.0, 0.0);
  }
}

// Deterministic two-phase reduction: part[b] = sum over a fixed stride of (off-diagonal |a|^2,
// all |a|^2); then one CTA adds the partials in order.
constexpr int JAC_RED_BLOCKS = 256;
__global__ void jacobi_offnorm_kernel(const double2* A, long long ld, int np, double* part) {
  __shared__ double so[256], st[256];
  double off = 0.0, tot = 0.0;
  const long long total = (long long)np * np;
  for (long long e = (long long)blockIdx.x * 256 + threadIdx.x; e < total; e += (long long)gridDim.x * 256) {
    const int i = (int)(e % np), j = (int)(e / np);
    const double2 v = A[(long long)i + (long long)j * ld];
    const double m = v.x * v.x + v.y * v.y;
    tot += m;
    if (i != j) off += m;
  }
  so[threadIdx.x] = off;
  st[threadIdx.x] = tot;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      so[threadIdx.x] += so[threadIdx.x + w];
      st[threadIdx.x] += st[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = so[0];
    part[2 * blockIdx.x + 1] = st[0];
  }
}
__global__ void jacobi_offnorm_final(const double* part, int nblk, double* out) {
  if (threadIdx.x == 0) {
    double off = 0.0, tot = 0.0;
    for (int b = 0; b < nblk; ++b) {
      off += part[2 * b];
      tot += part[2 * b + 1];
    }
    out[0] = off;
    out[1] = tot;
  }
}

// Eigenvalues (real diagonal) to a dense vector.
__global__ void jacobi_diag_kernel(const double2* A, long long ld, int np, double* w) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < np) w[i] = A[(long long)i + (long long)i * ld].x;
}

// Y columns in sorted order: Ys[:, k] = Y[:, order[k]], rows [0, n).  Real output takes the real
// part (the real symmetric problem runs through the complex solver with e = +-1: imaginary parts
// stay exactly zero).
template <typename T>
__global__ void jacobi_gather_kernel(const double2* Y, long long ld, int n, const int* order, T* Ys,
                                     long long lds);
template <>
__global__ void jacobi_gather_kernel<double2>(const double2* Y, long long ld, int n, const int* order,
                                              double2* Ys, long long lds) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)n * n) return;
  const int i = (int)(e % n), k = (int)(e / n);
  Ys[(long long)i + (long long)k * lds] = Y[(long long)i + (long long)order[k] * ld];
}
template <>
__global__ void jacobi_gather_kernel<double>(const double2* Y, long long ld, int n, const int* order,
                                             double* Ys, long long lds) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)n * n) return;
  const int i = (int)(e % n), k = (int)(e / n);
  Ys[(long long)i + (long long)k * lds] = Y[(long long)i + (long long)order[k] * ld].x;
}

// Real quotient into the complex solver buffer.
__global__ void real_to_complex_kernel(const double* Ar, long long ldr, double2* A, long long ld, int n) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)n * n) return;
  const int i = (int)(e % n), j = (int)(e / n);
  A[(long long)i + (long long)j * ld] = make_double2(Ar[(long long)i + (long long)j * ldr], 0.0);
}

}  // namespace chase
