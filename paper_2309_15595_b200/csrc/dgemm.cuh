// dgemm.cuh -- real-double tensor-core GEMM with the fused Chebyshev-recurrence epilogue, the
// real-symmetric counterpart of zgemm.cuh (SYMM of the filter for real problems, P:76
// "templated for complex/real type"; BASELINE config C5).
//
//   out[m, n] = alpha * ( sum_k opA[m, k] * X[k, n] - c * band(xin)[m, n] ) + beta * out[m, n]
//
// Same pipeline as zgemm (TMA + 128B swizzle, mbarrier ring refilled by thread 0, 8 DMMA
// warps).  Tiles: 128 x 128 outputs per CTA, 16 k per stage (one 128-byte row),
// 32 x 64 per warp.  Inside each stage the four m16n8k4 sub-steps h use the XOR-linear k
// permutation k = (t&1 ? 3 : 0) ^ (t&2 ? 12 : 0) ^ (h&1 ? 1 : 0) ^ (h&2 ? 4 : 0)
// (t = lane%4), chosen by exhaustive search so every 64-bit fragment load of A, A^T and X is
// bank-conflict free under the swizzle.
#pragma once
#include "common.cuh"

namespace chase {

#ifndef DG_BM_
#define DG_BM_ 128
#endif
#ifndef DG_BN_
#define DG_BN_ 128
#endif
constexpr int DG_BM = DG_BM_;
constexpr int DG_BN = DG_BN_;
constexpr int DG_BK = 16;
constexpr int DG_WM = DG_BM / 4;                 // warp tile rows (4 warps along M)
constexpr int DG_WN = DG_BN / 2;                 // warp tile cols (2 warps along N)
constexpr int DG_MT = DG_WM / 16;                // m16 tiles per warp
constexpr int DG_NT = DG_WN / 8;                 // n8 tiles per warp
constexpr int DG_STAGES = 196608 / ((DG_BM + DG_BN) * DG_BK * 8);
constexpr int DG_GROUP_M = 8;      // m-tiles per raster group
constexpr int DG_CONSUMERS = 8;   // 4 along M x 2 along N
constexpr int DG_THREADS = DG_CONSUMERS * 32;   // no dedicated producer warp: 9 warps would cap registers at 168
constexpr int DG_A_BYTES = DG_BM * DG_BK * 8;
constexpr int DG_X_BYTES = DG_BN * DG_BK * 8;
constexpr int DG_STAGE_BYTES = DG_A_BYTES + DG_X_BYTES;
constexpr int DG_SMEM_BYTES = DG_STAGES * DG_STAGE_BYTES + 1024 + 2 * DG_STAGES * 8;
#ifndef DG_BN_NARROW_
#define DG_BN_NARROW_ 32
#endif
constexpr int DG_BN_NARROW = DG_BN_NARROW_;  // remainder-column tile width (see dgemm_kernel)
// dgemm_kernel stages hold DG_KS k-slabs of DG_BK (one 128-byte swizzle row of k each, one TMA box
// per operand and slab): a k-tile is DG_BKT = DG_KS * DG_BK deep, so the per-k-tile barrier and
// refill work is spread over DG_KS times more DMMAs (the fused kernel keeps one slab per stage).
#ifndef DG_KSUB
#define DG_KSUB 2
#endif
constexpr int DG_KS = DG_KSUB;
constexpr int DG_BKT = DG_KS * DG_BK;
__host__ __device__ constexpr int dg_stages(int bn) { return 196608 / ((DG_BM + bn) * DG_BKT * 8); }
__host__ __device__ constexpr int dg_smem_bytes(int bn) {
  return dg_stages(bn) * (DG_BM + bn) * DG_BKT * 8 + 1024 + 2 * dg_stages(bn) * 8;
}

struct DGemmArgs {
  int M, N, K;
  int a_d0, a_d1;
  int x_k0, x_n0;
  double* out;
  long long ldo;
  const double* xin;
  long long ldx;
  double alpha, beta, c;
  int use_beta;
  int band_lo, band_hi;
  int band_shift;
  int upper_only;
  const int* abort_flag;
  const int* band_map;     // non-null (block-cyclic): see zgemm.cuh
  int diag_k;              // block-diagonal k ranges: see zgemm.cuh
  int a3d;                 // NoTrans only: tmA is the 3D view {16 doubles, k, m/16} -> 1 TMA/stage
  const double* col_shift; // non-null: out -= col_shift[n] * y2(m, n) before alpha (Alg.2 l.25)
  const double* y2;
  long long ldy2;
  int k_split;             // split-K: see zgemm.cuh
  long long split_ld;
  int tail_tiles;          // split-K tail of a big GEMM: see zgemm.cuh
  int tile_offset;
  int tri_k;               // X upper triangular: see zgemm.cuh
  int bat_a, bat_x;        // batched launch: see zgemm.cuh
  long long bat_out;
};

__device__ __forceinline__ int dg_kperm(int t, int h) {
  return ((t & 1) ? 3 : 0) ^ ((t & 2) ? 12 : 0) ^ ((h & 1) ? 1 : 0) ^ ((h & 2) ? 4 : 0);
}

// SPLIT (compile time): split-K variant (k_split > 1); the default instantiation is the plain
// GEMM with no split arithmetic in its hot loop.  BN_ (compile time): output columns per CTA --
// DG_BN for the bulk of a GEMM, DG_BN_NARROW for the N mod DG_BN remainder columns (a ragged
// width pads to 32, not 128, columns; the ramp-degree steps of C5 wasted 3.8 % of their DMMA
// work on padding with 128-wide tiles only).
template <bool TRANS, bool SPLIT = false, int BN_ = DG_BN, bool EXT = false>
__global__ void __launch_bounds__(DG_THREADS, 1)
    dgemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX,
                 const DGemmArgs g) {
  constexpr int WN_ = BN_ / 2, NT_ = WN_ / 8;                     // warp tile columns, n8 tiles
  constexpr int SLA = DG_BM * DG_BK * 8, SLX = BN_ * DG_BK * 8;   // one k-slab of A / X
  constexpr int AB_ = DG_KS * SLA, SB_ = DG_KS * (SLA + SLX), ST_ = dg_stages(BN_);
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment for the 128B swizzle, derived from the __shared__ array so every
  // fragment load stays an LDS (a pointer rebuilt from an integer becomes a generic LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST_ * SB_);
  uint64_t* empty = full + ST_;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grouped rasterisation (1D grid): consecutive CTAs walk DG_GROUP_M m-tiles, then the next
  // n-tile, so the CTAs resident at one time share A rows and X columns in L2
  const int n_tiles = (g.N + BN_ - 1) / BN_, m_tiles = (g.M + DG_BM - 1) / DG_BM;
  // split-K: the grid holds k_split copies of the tile grid, copy s sums its own k range
  const int tiles_launch = SPLIT && g.tail_tiles > 0 ? g.tail_tiles : n_tiles * m_tiles;
  const int split = SPLIT ? (int)blockIdx.x / tiles_launch : 0;
  const unsigned bid = SPLIT ? (unsigned)(g.tile_offset * (g.tail_tiles > 0) + (int)blockIdx.x - split * tiles_launch)
                             : blockIdx.x;
  const int group = bid / (DG_GROUP_M * n_tiles);
  const int first_m = group * DG_GROUP_M;
  const int gm = min(DG_GROUP_M, m_tiles - first_m);
  const int within = bid - group * DG_GROUP_M * n_tiles;
  const int m0 = (first_m + within % gm) * DG_BM;
  const int n0 = (EXT && g.tri_k ? n_tiles - 1 - within / gm : within / gm) * BN_;
  if (g.upper_only && m0 > n0 + BN_ - 1) return;
  if (g.abort_flag != nullptr && *g.abort_flag != 0) return;
  const int Kt = EXT && g.tri_k ? min(g.K, n0 + BN_) : g.K;   // K of this tile
  const int KT_all = (Kt + DG_BKT - 1) / DG_BKT;
  const int KTc = SPLIT ? (KT_all + g.k_split - 1) / g.k_split : KT_all;
  const int KT = min(KTc, KT_all - split * KTc);   // >= 1: the host never launches an empty split
  const int kbase = split * KTc * DG_BKT;
  const int Krem = Kt - kbase;                     // K left from this split's first k
  const int bz = EXT ? (int)blockIdx.y : 0;       // batch index (EXT: batched launches)
  const int a_d0 = g.a_d0 + bz * g.bat_a, a_d1 = g.a_d1 + bz * g.bat_a;
  const int x_k0 = g.x_k0 + bz * g.bat_x, x_n0 = g.x_n0 + bz * g.bat_x;
  double* const gout = g.out + bz * g.bat_out;
  const int dk = (g.diag_k == 1 ? n0 : (g.diag_k == 2 ? m0 : 0)) + kbase;   // per-CTA k offset

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST_; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], DG_CONSUMERS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // stage `s` <- k-tile `kt` (TMA, completion on full[s]); issued by thread 0 only
  auto issue = [&](int kt, int s) {
    mbar_arrive_expect_tx(&full[s], SB_);
#pragma unroll
    for (int u = 0; u < DG_KS; ++u) {
      uint8_t* sa = smem + s * SB_ + u * SLA;
      uint8_t* sx = smem + s * SB_ + AB_ + u * SLX;
      const int k0 = kt * DG_BKT + u * DG_BK + dk;
      if (TRANS) {
        tma_load_2d(sa, &tmA, a_d0 + k0, a_d1 + m0, &full[s]);     // box 16 k x 128 m
      } else {
        if (g.a3d) {
          tma_load_3d(sa, &tmA, 0, a_d1 + k0, (a_d0 + m0) / 16, &full[s]);
        } else {
#pragma unroll
          for (int b = 0; b < DG_BM / 16; ++b)                    // box 16 m x 16 k
            tma_load_2d(sa + b * 2048, &tmA, a_d0 + m0 + 16 * b, a_d1 + k0, &full[s]);
        }
      }
      tma_load_2d(sx, &tmX, x_k0 + k0, x_n0 + n0, &full[s]);       // box 16 k x BN n
    }
  };
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmX);
    for (int kt = 0; kt < ST_ && kt < KT; ++kt) issue(kt, kt);
  }

  const int wm = warp & 3, wn = warp >> 2;
  const int gq = lane >> 2, tq = lane & 3;
  double acc[DG_MT][NT_][4];
#pragma unroll
  for (int i = 0; i < DG_MT; ++i)
#pragma unroll
    for (int j = 0; j < NT_; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;

  // fragments double-buffered across sub-steps and k-tiles (see zgemm.cuh)
  constexpr int SUBS = DG_BKT / 4;
  struct Frag {
    double a[DG_MT][2], b[NT_];
  };
  auto load = [&](Frag& f, int kt, int sub) {
    const int u = sub >> 2, h = sub & 3;
    const int k = dg_kperm(tq, h);
    const uint8_t* sa = smem + (kt % ST_) * SB_ + u * SLA;
    const uint8_t* sx = smem + (kt % ST_) * SB_ + AB_ + u * SLX;
#pragma unroll
    for (int mt = 0; mt < DG_MT; ++mt)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int m = wm * DG_WM + mt * 16 + r * 8 + gq;
        const int off = TRANS ? m * 128 + ((((k >> 1) ^ gq) << 4) | ((k & 1) << 3))
                              : (m >> 4) * 2048 + k * 128 +
                                    (((((m & 15) >> 1) ^ (k & 7)) << 4) | ((m & 1) << 3));
        f.a[mt][r] = *reinterpret_cast<const double*>(sa + off);
      }
#pragma unroll
    for (int nt = 0; nt < NT_; ++nt) {
      const int n = wn * WN_ + nt * 8 + gq;
      f.b[nt] = *reinterpret_cast<const double*>(sx + n * 128 + ((((k >> 1) ^ gq) << 4) | ((k & 1) << 3)));
    }
    if (kt * DG_BKT + u * DG_BK + k >= Krem) {
#pragma unroll
      for (int mt = 0; mt < DG_MT; ++mt) f.a[mt][0] = f.a[mt][1] = 0.0;
#pragma unroll
      for (int nt = 0; nt < NT_; ++nt) f.b[nt] = 0.0;
    }
  };
  Frag cur, nxt;
  mbar_wait(&full[0], 0);
  load(cur, 0, 0);
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % ST_;
#pragma unroll
    for (int sub = 0; sub < SUBS; ++sub) {
      if (sub + 1 < SUBS) {
        load(nxt, kt, sub + 1);
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (kt + 1 < KT) {
          mbar_wait(&full[(kt + 1) % ST_], ((kt + 1) / ST_) & 1);
          load(nxt, kt + 1, 0);
        }
      }
#pragma unroll
      for (int mt = 0; mt < DG_MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT_; ++nt) dmma_16x8x4(acc[mt][nt], cur.a[mt][0], cur.a[mt][1], cur.b[nt]);
      cur = nxt;
    }
    // refill the stage released one iteration ago (most likely already drained by all warps)
    // the refill duty rotates over the warps so no single warp carries the producer work
    if (lane == 0 && warp == (kt & (DG_CONSUMERS - 1)) && kt >= 1 && kt - 1 + ST_ < KT) {
      const int sp = (kt - 1) % ST_;
      mbar_wait(&empty[sp], ((kt - 1) / ST_) & 1);
      issue(kt - 1 + ST_, sp);
    }
  }

#pragma unroll
  for (int mt = 0; mt < DG_MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT_; ++nt)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int row = m0 + wm * DG_WM + mt * 16 + gq + ((r & 2) ? 8 : 0);
        const int col = n0 + wn * WN_ + nt * 8 + 2 * tq + (r & 1);
        if (row < g.M && col < g.N) {
          double v = acc[mt][nt][r];
          const int bsrc = g.band_map != nullptr ? g.band_map[row]
                           : (row >= g.band_lo && row < g.band_hi ? row + g.band_shift : -1);
          if (bsrc >= 0) v -= g.c * g.xin[(long long)bsrc + (long long)col * g.ldx];
          if (g.col_shift != nullptr) v -= g.col_shift[col] * g.y2[(long long)row + (long long)col * g.ldy2];
          v *= g.alpha;
          double* o = SPLIT && g.tail_tiles > 0
                           ? gout + ((long long)split * g.tail_tiles + (long long)(bid - g.tile_offset)) * (DG_BM * BN_) +
                                 (row - m0) + (long long)(col - n0) * DG_BM
                           : gout + (long long)split * g.split_ld + (long long)row + (long long)col * g.ldo;
          if (g.use_beta) v += g.beta * *o;
          *o = v;
        }
      }
}

}  // namespace chase
