// zgemm.cuh -- complex-double tensor-core GEMM with the Chebyshev-recurrence epilogue fused
// (the HEMM of the filter; also the Gram / trailing updates of CholeskyQR, Alg.3).
//
//   out[m, n] = alpha * ( sum_k opA[m, k] * X[k, n]  -  c * band(xin)[m, n] ) + beta * out[m, n]
//
// opA = A (NoTrans, even filter steps "H^H B -> C") or A^H (ConjTrans, odd steps "H C -> B",
// P:149), A read through a TMA tensor map, never modified.  band(xin) is non-zero only on rows
// [band_lo, band_hi) -- the diagonal rows of -cI this rank owns (reading #6); the beta term is
// applied only when use_beta (designated rank, reading #7; never on step 1 so B is never read
// before it is written).
//
// B200 design: FP64 has no tcgen05 kind, so the math runs on the FP64 tensor pipe through
// warp-level DMMA (mma.sync.m16n8k4.f64, 37.1 TFLOP/s measured).  Operand tiles are staged by
// TMA (cp.async.bulk.tensor, SWIZZLE_128B) into an 8-stage mbarrier ring; thread 0 issues the
// TMA loads in-line (a 9th producer warp would put 3 warps on one SM sub-partition and cap
// registers at 168 -> spills); 8 DMMA warps each own a 32x32 complex sub-tile (the complex
// product is split into 4 real DMMA products, 8 real flops per complex MAC).
// The k index inside each 8-wide smem row is permuted (k = 2t + h for mma sub-step h) so every
// 128-bit fragment load of A, A^H and X is bank-conflict free under the 128-byte swizzle.
#pragma once
#include "common.cuh"

namespace chase {

constexpr int ZG_BM = 128;        // rows of out per CTA
constexpr int ZG_BN = 64;         // columns of out per CTA
#ifndef ZG_KSUB
#define ZG_KSUB 2                 // 8-wide k slabs (one 128-byte swizzle row each) per stage
#endif
constexpr int ZG_KS = ZG_KSUB;
constexpr int ZG_BK = 8 * ZG_KS;  // complex k per stage
constexpr int ZG_STAGES = 8 / ZG_KS;
constexpr int ZG_GROUP_M = 8;      // m-tiles per raster group
#ifndef ZG_WARPS_N
#define ZG_WARPS_N 2              // warps along N (4 along M)
#endif
constexpr int ZG_WNW = ZG_WARPS_N;
constexpr int ZG_CONSUMERS = 4 * ZG_WNW;          // consumer warps
constexpr int ZG_WN = ZG_BN / ZG_WNW;             // warp tile columns
constexpr int ZG_NT = ZG_WN / 8;                  // n8 tiles per warp
#ifndef ZG_WS
#define ZG_WS 0                   // 1: producer warpgroup + setmaxnreg (warp specialisation)
#endif
// ZG_WS == 0: no dedicated producer warp (9 warps would cap registers at 168); the refill duty
// rotates over the 8 MMA warps.  ZG_WS == 1: a 4-warp producer group drops to 40 registers with
// setmaxnreg and the two MMA warpgroups rise to 232.
constexpr int ZG_THREADS = (ZG_CONSUMERS + (ZG_WS ? 4 : 0)) * 32;
constexpr int ZG_A_SLAB = ZG_BM * 8 * 16;       // 16 KB per 8-wide k slab
constexpr int ZG_X_SLAB = ZG_BN * 8 * 16;       // 8 KB per 8-wide k slab
constexpr int ZG_A_BYTES = ZG_A_SLAB * ZG_KS;
constexpr int ZG_X_BYTES = ZG_X_SLAB * ZG_KS;
constexpr int ZG_STAGE_BYTES = ZG_A_BYTES + ZG_X_BYTES;
constexpr int ZG_SMEM_BYTES = ZG_STAGES * ZG_STAGE_BYTES + 1024 + 2 * ZG_STAGES * 8;
constexpr int ZG_BN_NARROW = 32;  // remainder-column tile width (see zgemm_kernel)
__host__ __device__ constexpr int zg_smem_bytes(int bn) { return ZG_STAGES * (ZG_A_BYTES + bn * 8 * 16 * ZG_KS) + 1024 + 2 * ZG_STAGES * 8; }

struct ZGemmArgs {
  int M, N, K;
  int a_d0, a_d1;          // tensor-map coordinate offsets of opA's (0,0) element, in complex
                           // elements: NoTrans (row = m, col = k), ConjTrans (row = k, col = m)
  int x_k0, x_n0;          // X tensor-map offsets (row = k, col = n)
  double2* out;            // out(m, n) = out[m + n * ldo]
  long long ldo;
  const double2* xin;      // band input: xin(row, n) = xin[row + n * ldx]
  long long ldx;
  double alpha, beta, c;
  int use_beta;
  int band_lo, band_hi;    // out rows [band_lo, band_hi) subtract c * xin[row + band_shift, n]
  int band_shift;
  int upper_only;          // skip CTAs whose tile lies strictly below the diagonal (m > n)
  const int* abort_flag;   // non-null: skip the whole GEMM when *abort_flag != 0 (POTRF info)
  int diag_k;              // block-diagonal right/left factor (Jacobi eigensolver updates):
                           //   1: the k range of n-tile n0 starts at n0; 2: of m-tile m0 at m0
  const int* band_map;     // non-null (block-cyclic): out row m subtracts c * xin[band_map[m], n]
                           //   when band_map[m] >= 0; replaces [band_lo, band_hi)
  int a3d;                 // NoTrans only: tmA is the 3D view {8 complex, k, m/8} -> 1 TMA/stage
  const double* col_shift; // non-null: out -= col_shift[n] * y2(m, n) before alpha (residual,
  const double2* y2;       //   Alg.2 l.25 "B <- B - ritzv B2" fused into the HEMM epilogue)
  long long ldy2;
  int k_split;             // > 1: split-K -- CTA blockIdx / tiles takes k-tiles [s KTc, (s+1) KTc)
  long long split_ld;      //   and writes its partial product to out + s * split_ld (no beta)
  int tail_tiles;          // SPLIT, > 0: the launch covers only tiles [tile_offset, +tail_tiles)
  int tile_offset;         //   of the raster (the wave-quantisation tail of a big GEMM), and each
                           //   partial tile is stored tile-local: out + (s tail_tiles + j) BM BN,
                           //   column-major with ld BM (gemm_tail_epilogue_kernel finishes them)
  int tri_k;               // X upper triangular (V R^{-1} of the TRSM): tile (m0, n0) sums only
                           //   k < min(K, n0 + BN); n-tiles rastered last-first (longest first)
  int bat_a, bat_x;        // batched launch (gridDim.y > 1, block-diagonal sub-problems of the
  long long bat_out;       //   recursive-doubling TRTRI): batch z adds z*bat_a to both A map
                           //   coordinates, z*bat_x to both X map coordinates, z*bat_out to out
};

// SPLIT (compile time): split-K variant (k_split > 1); the default instantiation is the plain
// GEMM with no split arithmetic in its hot loop.  BN_ (compile time): output columns per CTA --
// ZG_BN for the bulk of a GEMM, ZG_BN_NARROW for the N mod ZG_BN remainder columns (so a
// ragged width pads to 32, not 64, columns; the X tensor map box must match).  EXT (compile
// time): the tri_k and batched modes of the TRSM / TRTRI; the filter instantiations leave them
// out (their prologue arithmetic cost the filter HEMM 0.6 %, measured A/B on one box).
template <bool CONJ, bool SPLIT = false, int BN_ = ZG_BN, bool EXT = false>
__global__ void __launch_bounds__(ZG_THREADS, 1)
    zgemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX,
                 const ZGemmArgs g) {
  constexpr int WN_ = BN_ / ZG_WNW, NT_ = WN_ / 8;               // warp tile columns, n8 tiles
  constexpr int XS_ = BN_ * 8 * 16, XB_ = XS_ * ZG_KS, SB_ = ZG_A_BYTES + XB_;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment for the 128B swizzle, derived from the __shared__ array so every
  // fragment load stays an LDS (a pointer rebuilt from an integer becomes a generic LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ZG_STAGES * SB_);
  uint64_t* empty = full + ZG_STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grouped rasterisation (1D grid): consecutive CTAs walk ZG_GROUP_M m-tiles, then the next
  // n-tile, so the CTAs resident at one time share A rows and X columns in L2
  const int n_tiles = (g.N + BN_ - 1) / BN_, m_tiles = (g.M + ZG_BM - 1) / ZG_BM;
  // split-K: the grid holds k_split copies of the tile grid, copy s sums its own k range
  const int tiles_launch = SPLIT && g.tail_tiles > 0 ? g.tail_tiles : n_tiles * m_tiles;
  const int split = SPLIT ? (int)blockIdx.x / tiles_launch : 0;
  const unsigned bid = SPLIT ? (unsigned)(g.tile_offset * (g.tail_tiles > 0) + (int)blockIdx.x - split * tiles_launch)
                             : blockIdx.x;
  const int group = bid / (ZG_GROUP_M * n_tiles);
  const int first_m = group * ZG_GROUP_M;
  const int gm = min(ZG_GROUP_M, m_tiles - first_m);
  const int within = bid - group * ZG_GROUP_M * n_tiles;
  const int m0 = (first_m + within % gm) * ZG_BM;
  const int n0 = (EXT && g.tri_k ? n_tiles - 1 - within / gm : within / gm) * BN_;
  if (g.upper_only && m0 > n0 + BN_ - 1) return;
  if (g.abort_flag != nullptr && *g.abort_flag != 0) return;
  const int Kt = EXT && g.tri_k ? min(g.K, n0 + BN_) : g.K;   // K of this tile
  const int KT_all = (Kt + ZG_BK - 1) / ZG_BK;
  const int KTc = SPLIT ? (KT_all + g.k_split - 1) / g.k_split : KT_all;
  const int KT = min(KTc, KT_all - split * KTc);   // >= 1: the host never launches an empty split
  const int kbase = split * KTc * ZG_BK;
  const int Krem = Kt - kbase;                     // K left from this split's first k
  const int bz = EXT ? (int)blockIdx.y : 0;       // batch index (EXT: batched launches)
  const int a_d0 = g.a_d0 + bz * g.bat_a, a_d1 = g.a_d1 + bz * g.bat_a;
  const int x_k0 = g.x_k0 + bz * g.bat_x, x_n0 = g.x_n0 + bz * g.bat_x;
  double2* const gout = g.out + bz * g.bat_out;
  const int dk = (g.diag_k == 1 ? n0 : (g.diag_k == 2 ? m0 : 0)) + kbase;   // per-CTA k offset

  if (threadIdx.x == 0) {
    for (int s = 0; s < ZG_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ZG_CONSUMERS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // stage `s` <- k-tile `kt` (TMA, completion on full[s]); issued by thread 0 only
  auto issue = [&](int kt, int s) {
    mbar_arrive_expect_tx(&full[s], SB_);
    uint8_t* sa = smem + s * SB_;
    uint8_t* sx = sa + ZG_A_BYTES;
#pragma unroll
    for (int u = 0; u < ZG_KS; ++u) {
      const int k0 = kt * ZG_BK + 8 * u + dk;
      uint8_t* sau = sa + u * ZG_A_SLAB;
      if (CONJ) {
        // opA[m][k] = conj(A[k][m]); A rows (k) contiguous: one 128 x 8 box, row = m
        tma_load_2d(sau, &tmA, 2 * (a_d0 + k0), a_d1 + m0, &full[s]);
      } else {
        // A rows (m) contiguous: 16 boxes of 8 m x 8 k, box b holds rows [8b, 8b+8), row = k
        if (g.a3d) {
          tma_load_3d(sau, &tmA, 0, a_d1 + k0, (a_d0 + m0) / 8, &full[s]);
        } else {
#pragma unroll
          for (int b = 0; b < ZG_BM / 8; ++b)
            tma_load_2d(sau + b * 1024, &tmA, 2 * (a_d0 + m0 + 8 * b), a_d1 + k0, &full[s]);
        }
      }
      tma_load_2d(sx + u * XS_, &tmX, 2 * (x_k0 + k0), x_n0 + n0, &full[s]);
    }
  };
#if ZG_WS
  if (warp < 4) {                                  // producer warpgroup
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == 0 && lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmX);
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % ZG_STAGES;
        if (kt >= ZG_STAGES) mbar_wait(&empty[s], ((kt / ZG_STAGES) & 1) ^ 1);
        issue(kt, s);
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
  const int cwarp = warp - 4;
#else
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmX);
    for (int kt = 0; kt < ZG_STAGES && kt < KT; ++kt) issue(kt, kt);
  }
  const int cwarp = warp;
#endif

  // -------------------------------------------------------------- consumer warps
  const int wm = cwarp & 3, wn = cwarp >> 2;
  const int gq = lane >> 2, tq = lane & 3;
  double acc_re[2][NT_][4], acc_im[2][NT_][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NT_; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc_re[i][j][r] = acc_im[i][j][r] = 0.0;

  // Fragments are double-buffered in registers: the loads of sub-step t+1 (including the first
  // sub-step of the next k-tile, after its full barrier) are issued before the DMMAs of t.
  constexpr int SUBS = 2 * ZG_KS;                      // m16n8k4 sub-steps per k-tile
  struct Frag {
    double2 a[2][2], b[NT_];
  };
  auto load = [&](Frag& f, int kt, int sub) {
    const int u = sub >> 1, h = sub & 1;
    const int k = 2 * tq + h;                          // k inside the 8-wide slab u
    const uint8_t* sa = smem + (kt % ZG_STAGES) * SB_ + u * ZG_A_SLAB;
    const uint8_t* sx = smem + (kt % ZG_STAGES) * SB_ + ZG_A_BYTES + u * XS_;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int m = wm * 32 + mt * 16 + r * 8 + gq;  // m & 7 == gq
        const int off = CONJ ? m * 128 + ((k ^ gq) << 4)
                             : (m >> 3) * 1024 + k * 128 + ((gq ^ k) << 4);
        f.a[mt][r] = *reinterpret_cast<const double2*>(sa + off);
      }
#pragma unroll
    for (int nt = 0; nt < NT_; ++nt) {
      const int n = wn * WN_ + nt * 8 + gq;
      f.b[nt] = *reinterpret_cast<const double2*>(sx + n * 128 + ((k ^ gq) << 4));
    }
    if (kt * ZG_BK + 8 * u + k >= Krem) {               // K tail (the TMA box may hold stale data)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) f.a[mt][0] = f.a[mt][1] = make_double2(0.0, 0.0);
#pragma unroll
      for (int nt = 0; nt < NT_; ++nt) f.b[nt] = make_double2(0.0, 0.0);
    }
  };
  auto mma = [&](const Frag& f) {
    // real parts of opA times X
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT_; ++nt) {
        dmma_16x8x4(acc_re[mt][nt], f.a[mt][0].x, f.a[mt][1].x, f.b[nt].x);
        dmma_16x8x4(acc_im[mt][nt], f.a[mt][0].x, f.a[mt][1].x, f.b[nt].y);
      }
    // imaginary parts: A: re -= Ai*Bi, im += Ai*Br;  A^H: re += Ai*Bi, im -= Ai*Br
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT_; ++nt) {
        const double bre = CONJ ? f.b[nt].y : -f.b[nt].y;
        const double bim = CONJ ? -f.b[nt].x : f.b[nt].x;
        dmma_16x8x4(acc_re[mt][nt], f.a[mt][0].y, f.a[mt][1].y, bre);
        dmma_16x8x4(acc_im[mt][nt], f.a[mt][0].y, f.a[mt][1].y, bim);
      }
  };

  Frag cur, nxt;
  mbar_wait(&full[0], 0);
  load(cur, 0, 0);
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % ZG_STAGES;
#pragma unroll
    for (int sub = 0; sub < SUBS; ++sub) {
      if (sub + 1 < SUBS) {
        load(nxt, kt, sub + 1);
      } else {
        // every fragment of stage s is in registers: release it, then prefetch the next tile
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (kt + 1 < KT) {
          mbar_wait(&full[(kt + 1) % ZG_STAGES], ((kt + 1) / ZG_STAGES) & 1);
          load(nxt, kt + 1, 0);
        }
      }
      mma(cur);
      cur = nxt;
    }
    // refill the stage released one iteration ago (most likely already drained by all warps)
    // the refill duty rotates over the warps so no single warp carries the producer work
    if (!ZG_WS && lane == 0 && warp == (kt & (ZG_CONSUMERS - 1)) && kt >= 1 && kt - 1 + ZG_STAGES < KT) {
      const int sp = (kt - 1) % ZG_STAGES;
      mbar_wait(&empty[sp], ((kt - 1) / ZG_STAGES) & 1);
      issue(kt - 1 + ZG_STAGES, sp);
    }
  }

  // -------------------------------------------------------------- fused recurrence epilogue
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT_; ++nt)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int row = m0 + wm * 32 + mt * 16 + gq + ((r & 2) ? 8 : 0);
        const int col = n0 + wn * WN_ + nt * 8 + 2 * tq + (r & 1);
        if (row < g.M && col < g.N) {
          double vr = acc_re[mt][nt][r], vi = acc_im[mt][nt][r];
          const int bsrc = g.band_map != nullptr ? g.band_map[row]
                           : (row >= g.band_lo && row < g.band_hi ? row + g.band_shift : -1);
          if (bsrc >= 0) {
            const double2 x = g.xin[(long long)bsrc + (long long)col * g.ldx];
            vr -= g.c * x.x;
            vi -= g.c * x.y;
          }
          if (g.col_shift != nullptr) {
            const double2 y = g.y2[(long long)row + (long long)col * g.ldy2];
            const double lam = g.col_shift[col];
            vr -= lam * y.x;
            vi -= lam * y.y;
          }
          vr *= g.alpha;
          vi *= g.alpha;
          double2* o = SPLIT && g.tail_tiles > 0
                           ? gout + ((long long)split * g.tail_tiles + (long long)(bid - g.tile_offset)) * (ZG_BM * BN_) +
                                 (row - m0) + (long long)(col - n0) * ZG_BM
                           : gout + (long long)split * g.split_ld + (long long)row + (long long)col * g.ldo;
          if (g.use_beta) {
            const double2 old = *o;
            vr += g.beta * old.x;
            vi += g.beta * old.y;
          }
          *o = make_double2(vr, vi);
        }
      }
}

}  // namespace chase
