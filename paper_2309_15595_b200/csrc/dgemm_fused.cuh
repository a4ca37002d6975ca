// dgemm_fused.cuh -- the real-symmetric filter step as ONE kernel (BASELINE C5 is real, P:76
// "templated for complex/real type"): the dgemm mainloop (dgemm.cuh: 128 x BN tiles, DG_KS
// 16-k slabs per stage, XOR-linear k permutation) inside the persistent push/owner/broadcast protocol of
// zgemm_fused.cuh (dynamic tile scheduler, partial tiles pushed into the owner's staging slots
// over NVLink, fixed-order owner sum + beta term, broadcast, delivery counters, bounded spins).
// See zgemm_fused.cuh for the protocol and its deadlock-freedom argument; only the element type
// and the tile mainloop differ.
#pragma once
#include "dgemm.cuh"
#include "zgemm_fused.cuh"

namespace chase {

template <bool TRANS, int BN_ = DG_BN>
__global__ void __launch_bounds__(DG_THREADS, 1)
    dgemm_fused_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX,
                       const DGemmArgs g, const FusedArgs f) {
  constexpr int WN_ = BN_ / 2, NT_ = WN_ / 8;                     // warp tile columns, n8 tiles
  constexpr int SLA = DG_BM * DG_BK * 8, SLX = BN_ * DG_BK * 8;   // one k-slab of A / X
  constexpr int AB_ = DG_KS * SLA, SB_ = DG_KS * (SLA + SLX), ST_ = dg_stages(BN_);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST_ * SB_);
  uint64_t* empty = full + ST_;
  __shared__ int s_abort;
  __shared__ int s_q[FUSED_QCAP];
  __shared__ int s_qh, s_qt, s_cmd;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = (g.N + BN_ - 1) / BN_, m_tiles = (g.M + DG_BM - 1) / DG_BM;
  const int T = f.tiles > 0 ? f.tiles : n_tiles * m_tiles;
  const int KT = (g.K + DG_BKT - 1) / DG_BKT;
  constexpr int RING = ST_ + 4;                  // see zgemm_fused.cuh (grab 2 ahead)
  __shared__ int s_tile[RING];
  auto grab = [&]() -> int {
    const unsigned long long v = atomicAdd(f.tile_ctr, 1ull) - f.ctr_base;
    return v < (unsigned long long)T ? (int)v : -1;
  };
  auto tile_origin = [&](int t, int& m0, int& n0) {
    const int group = t / (DG_GROUP_M * n_tiles);
    const int first_m = group * DG_GROUP_M;
    const int gm = min(DG_GROUP_M, m_tiles - first_m);
    const int within = t - group * DG_GROUP_M * n_tiles;
    m0 = (first_m + within % gm) * DG_BM;
    n0 = (within / gm) * BN_;
  };

  if (threadIdx.x == 0) {
    s_abort = 0;
    s_qh = s_qt = 0;
    const long long t0 = clock64();
    while (ld_acquire_sys_u64(f.done[f.me]) < f.done_target) {
      __nanosleep(256);
      if (clock64() - t0 > FUSED_SPIN_CYCLES) {
        printf("[chase fused] member %d CTA %d: previous step not delivered (%llu < %llu)\n", f.me,
               (int)blockIdx.x, ld_acquire_sys_u64(f.done[f.me]), f.done_target);
        atomicExch(f.err, 1);
        s_abort = 1;
        break;
      }
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
    for (int s = 0; s < ST_; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], DG_CONSUMERS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (s_abort) return;

  auto issue = [&](int q, int s) {
    if ((q + 2) % KT == 0) {
      const int sq = (q + 2) / KT;
      s_tile[sq % RING] = grab();
    }
    const int t = s_tile[(q / KT) % RING];
    if (t < 0) {
      mbar_arrive(&full[s]);
      return;
    }
    int m0, n0;
    tile_origin(t, m0, n0);
    mbar_arrive_expect_tx(&full[s], SB_);
#pragma unroll
    for (int u = 0; u < DG_KS; ++u) {
      const int k0 = (q % KT) * DG_BKT + u * DG_BK;
      uint8_t* sa = smem + s * SB_ + u * SLA;
      uint8_t* sx = smem + s * SB_ + AB_ + u * SLX;
      if (TRANS) {
        tma_load_2d(sa, &tmA, g.a_d0 + k0, g.a_d1 + m0, &full[s]);
      } else if (g.a3d) {
        tma_load_3d(sa, &tmA, 0, g.a_d1 + k0, (g.a_d0 + m0) / 16, &full[s]);
      } else {
#pragma unroll
        for (int b = 0; b < DG_BM / 16; ++b)
          tma_load_2d(sa + b * 2048, &tmA, g.a_d0 + m0 + 16 * b, g.a_d1 + k0, &full[s]);
      }
      tma_load_2d(sx, &tmX, g.x_k0 + k0, g.x_n0 + n0, &full[s]);
    }
  };
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmX);
    for (int sq = 0; sq * KT < 2; ++sq) s_tile[sq % RING] = grab();
    for (int gs = 0; gs < ST_; ++gs) issue(gs, gs);
  }

  const int wm = warp & 3, wn = warp >> 2;
  const int gq = lane >> 2, tq = lane & 3;
  double acc[DG_MT][NT_][4];
  auto zero_acc = [&]() {
#pragma unroll
    for (int i = 0; i < DG_MT; ++i)
#pragma unroll
      for (int j = 0; j < NT_; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;
  };
  zero_acc();

  constexpr int SUBS = DG_BKT / 4;
  struct Frag {
    double a[DG_MT][2], b[NT_];
  };
  auto load = [&](Frag& fr, int st, int kt, int sub) {    // st: smem stage
    const int u = sub >> 2, hsub = sub & 3;
    const int k = dg_kperm(tq, hsub);
    const uint8_t* sa = smem + st * SB_ + u * SLA;
    const uint8_t* sx = smem + st * SB_ + AB_ + u * SLX;
#pragma unroll
    for (int mt = 0; mt < DG_MT; ++mt)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int m = wm * DG_WM + mt * 16 + r * 8 + gq;
        const int off = TRANS ? m * 128 + ((((k >> 1) ^ gq) << 4) | ((k & 1) << 3))
                              : (m >> 4) * 2048 + k * 128 +
                                    (((((m & 15) >> 1) ^ (k & 7)) << 4) | ((m & 1) << 3));
        fr.a[mt][r] = *reinterpret_cast<const double*>(sa + off);
      }
#pragma unroll
    for (int nt = 0; nt < NT_; ++nt) {
      const int n = wn * WN_ + nt * 8 + gq;
      fr.b[nt] = *reinterpret_cast<const double*>(sx + n * 128 + ((((k >> 1) ^ gq) << 4) | ((k & 1) << 3)));
    }
    if (kt * DG_BKT + u * DG_BK + k >= g.K) {
#pragma unroll
      for (int mt = 0; mt < DG_MT; ++mt) fr.a[mt][0] = fr.a[mt][1] = 0.0;
#pragma unroll
      for (int nt = 0; nt < NT_; ++nt) fr.b[nt] = 0.0;
    }
  };

  // owner side: fixed-order sum of the m partial tiles of t (local slots), + beta V_{s-2},
  // broadcast into every member's output, delivery counters bumped
  auto reduce = [&](int t) {
    int m0, n0;
    tile_origin(t, m0, n0);
    double* const* outs = reinterpret_cast<double* const*>(f.out);
    const double* __restrict__ mine = reinterpret_cast<const double*>(f.P[f.me]);
    // row pairs as double2 (ldP, ldo and slot are even, every column 16-byte aligned; the pair
    // partner of an odd M's last row is padding, loaded and never stored): 64 BN_ pairs per tile,
    // up to 16 per thread per batch, all their loads in flight together
    constexpr int HM = DG_BM / 2;
    constexpr int PER2 = HM * BN_ / DG_THREADS;       // 32 (BN 128) or 8 (BN 32)
    constexpr int BATCH2 = PER2 < 16 ? PER2 : 16;
#pragma unroll 1
    for (int b0 = 0; b0 < PER2; b0 += BATCH2) {
      double2 sum[BATCH2];
#pragma unroll
      for (int i = 0; i < BATCH2; ++i) {
        const int e = threadIdx.x + (b0 + i) * DG_THREADS;
        const int row = m0 + 2 * (e % HM), col = n0 + e / HM;
        sum[i] = make_double2(0.0, 0.0);
        if (row < g.M && col < g.N) {
          const long long ip = (long long)row + (long long)(f.col_base + col) * f.ldP;
          sum[i] = *reinterpret_cast<const double2*>(mine + ip);
          for (int src = 1; src < f.m; ++src) {
            const double2 v = *reinterpret_cast<const double2*>(mine + (long long)src * f.slot + ip);
            sum[i].x += v.x;
            sum[i].y += v.y;
          }
          if (f.owner_beta) {
            const double2 old = *reinterpret_cast<const double2*>(outs[f.me] + (long long)row + (long long)col * g.ldo);
            sum[i].x += g.beta * old.x;
            sum[i].y += g.beta * old.y;
          }
        }
      }
#pragma unroll
      for (int i = 0; i < BATCH2; ++i) {
        const int e = threadIdx.x + (b0 + i) * DG_THREADS;
        const int row = m0 + 2 * (e % HM), col = n0 + e / HM;
        if (row >= g.M || col >= g.N) continue;
        const long long io = (long long)row + (long long)col * g.ldo;
        if (row + 1 < g.M) {
          for (int dst = 0; dst < f.m; ++dst) *reinterpret_cast<double2*>(outs[dst] + io) = sum[i];
        } else {
          for (int dst = 0; dst < f.m; ++dst) outs[dst][io] = sum[i].x;
        }
      }
    }
    // the CTA's stores happen before thread 0's system fence (bar.sync), which publishes them
    // all before the counters move (one fence per CTA, not one per thread)
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int dst = 0; dst < f.m; ++dst) atomicAdd_system(f.done[dst], 1ull);
    }
  };

  // Owned tiles wait in a small queue and are reduced as soon as all m partials are in, checked
  // (without blocking) after every tile; the CTA blocks only when the queue is full and, at the
  // end, until its queue is drained.  A straggling peer therefore never stalls the tensor pipe of
  // an owner that still has tiles to compute.
  auto flags_ready = [&](int t) -> bool {      // thread 0
    for (int src = 0; src < f.m; ++src)
      if (ld_acquire_sys_u32(f.flags[f.me] + (long long)(f.tile_base + t) * f.m + src) != f.ep) return false;
    return true;
  };
  auto drain = [&](bool final_) {
    for (;;) {
      if (threadIdx.x == 0) {
        int cmd = -1;
        if (s_qh < s_qt) {
          const int t = s_q[s_qh % FUSED_QCAP];
          bool ok = flags_ready(t);
          if (!ok && (final_ || s_qt - s_qh >= FUSED_QCAP)) {
            const long long t0 = clock64();
            while (!(ok = flags_ready(t))) {
              __nanosleep(64);
              if (clock64() - t0 > FUSED_SPIN_CYCLES) {
                printf("[chase fused] member %d CTA %d: tile %d partials missing (m %d, ep %u, flags %u %u, final %d, q %d..%d)\n",
                       f.me, (int)blockIdx.x, t, f.m, f.ep, f.flags[f.me][(long long)(f.tile_base + t) * f.m],
                       f.flags[f.me][(long long)(f.tile_base + t) * f.m + (f.m > 1 ? 1 : 0)], (int)final_, s_qh, s_qt);
                atomicExch(f.err, 1);
                s_abort = 1;
                break;
              }
            }
          }
          if (ok) {
            cmd = t;
            ++s_qh;
          }
        }
        s_cmd = cmd;
      }
      __syncthreads();
      const int t = s_cmd;
      __syncthreads();                         // s_cmd read by all before thread 0 rewrites it
      if (t < 0 || s_abort) return;
      reduce(t);
    }
  };

  auto epilogue = [&](int t) {
    int m0, n0;
    tile_origin(t, m0, n0);
    double* const* outs = reinterpret_cast<double* const*>(f.out);
    if (f.plain) {
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
              if (row >= g.band_lo && row < g.band_hi)
                v -= g.c * g.xin[(long long)(row + g.band_shift) + (long long)col * g.ldx];
              v *= g.alpha;
              double* o = outs[f.me] + (long long)row + (long long)col * g.ldo;
              if (f.owner_beta) v += g.beta * *o;
              *o = v;
            }
          }
      if (threadIdx.x == 0) atomicAdd(f.done[f.me], 1ull);
      return;
    }
    const int owner = (f.tile_base + t) % f.m;
    double* slot = reinterpret_cast<double*>(f.P[owner]) + (long long)f.me * f.slot;
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
            slot[(long long)row + (long long)(f.col_base + col) * f.ldP] = v * g.alpha;
          }
        }
    __syncthreads();                           // then one system release by thread 0
    if (threadIdx.x == 0) st_release_sys_u32(f.flags[owner] + (long long)(f.tile_base + t) * f.m + f.me, f.ep);
    if (threadIdx.x == 0 && owner == f.me) {       // reduce it later, without blocking now
      s_q[s_qt % FUSED_QCAP] = t;
      ++s_qt;
    }
    drain(false);
  };

  Frag cur, nxt;
  mbar_wait_dbg(&full[0], 0, 1, 0);
  int tile = s_tile[0];
  if (tile < 0) return;
  load(cur, 0, 0, 0);
  // stage and phase of issue index gs kept incrementally (ST_ = 3 for the wide tile: a division
  // per k-tile otherwise sits in front of every k-tile's first MMAs)
  int seq = 0, kt = 0, gs = 0, stg = 0, ph = 0;
  for (;;) {
    const int s = stg;
    const int stn = stg + 1 == ST_ ? 0 : stg + 1;         // stage / phase of gs + 1
    const int phn = stg + 1 == ST_ ? ph ^ 1 : ph;
    int next_tile = tile;
#pragma unroll
    for (int sub = 0; sub < SUBS; ++sub) {
      if (sub + 1 < SUBS) {
        load(nxt, s, kt, sub + 1);
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        mbar_wait_dbg(&full[stn], phn, 2, gs);
        if (kt + 1 < KT) {
          load(nxt, stn, kt + 1, 0);
        } else {
          next_tile = s_tile[(seq + 1) % RING];
          if (next_tile >= 0) load(nxt, stn, 0, 0);
        }
      }
#pragma unroll
      for (int mt = 0; mt < DG_MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT_; ++nt) dmma_16x8x4(acc[mt][nt], cur.a[mt][0], cur.a[mt][1], cur.b[nt]);
      cur = nxt;
    }
    if (lane == 0 && warp == (gs & (DG_CONSUMERS - 1)) && gs >= 1) {
      const int sp = stg == 0 ? ST_ - 1 : stg - 1;           // stage / phase of gs - 1
      mbar_wait_dbg(&empty[sp], stg == 0 ? ph ^ 1 : ph, 3, gs);
      issue(gs - 1 + ST_, sp);
    }
    ++gs;
    stg = stn;
    ph = phn;
    if (++kt == KT) {
      epilogue(tile);
      zero_acc();
      if (s_abort) {
        if (threadIdx.x == 0)
          for (int r = gs; r < gs + ST_ - 1; ++r) mbar_wait(&full[r % ST_], (r / ST_) & 1);
        return;
      }
      kt = 0;
      ++seq;
      tile = next_tile;
      if (tile < 0) break;
    }
  }
  drain(true);                                 // the owned tiles still waiting
}

}  // namespace chase
