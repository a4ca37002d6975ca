// zgemm_fused.cuh -- the filter step as ONE kernel: tensor-core HEMM + the AllReduce of its
// result over the reducing communicator, done tile by tile over NVLink peer memory.
//
// A filter step on a p x q grid is "partial_r = alpha (A_r^(H) X - c band) on every member r of
// the row (even step) / column (odd step) communicator, then AllReduce(SUM)" (Alg.2 l.12).
// Here every member runs a persistent grid (one CTA per SM) over the step's output tiles, handed
// out by a local dynamic tile scheduler.  After the K loop of output tile t a CTA
//   1. pushes its partial tile into its slot of the tile owner's staging area (NVLink stores;
//      owner = t mod m: the tiles in flight at any moment (consecutive ids from the dynamic
//      scheduler) spread their partials and broadcasts over all members' NVLink ports),
//   2. releases a per-(tile, member) arrival flag in the owner's memory,
// and, if it owns t, queues t.  After every tile the CTA checks its queue without blocking: an
// owned tile whose m flags are in is reduced -- the m partial tiles summed from its LOCAL slots
// in fixed member order (deterministic, identical bits on every member), + beta * V_{s-2}
// (replicated, read locally), pushed into the output buffer of every member, each member's
// delivery counter bumped.  The CTA blocks only when its queue is full or at the end of its tile
// stream, so a slower peer does not stall the owner's tensor pipe.  The next step's kernel waits
// until its delivery counter covers the whole previous step.  The reduction traffic of tile t
// overlaps the math of the tiles that follow it -- no separate collective launch.  Staging
// slots and flags are separate per step parity: a rank's row and column communicators progress
// independently, so a peer already in step s+1 must not touch what this rank still reads for s.
//
// The k-tile loads are refilled by the MMA warps in rotation (no producer warp); the tile id of
// each sequence position is grabbed from the scheduler two issue indices ahead.
// Deadlock freedom: all CTAs are co-resident (grid <= #SMs, 1 CTA/SM); a partial is always
// published before its producer waits on anything; a blocked CTA waits on a tile no later than
// its current one while every tile it holds ahead (prefetched) is later, so every chain of waits
// decreases in tile index and ends at a CTA that is still computing.
// Every spin is bounded (~10 s at 2 GHz); on timeout the kernel sets *err and gives up so a
// broken peer can never hang the GPU.
#pragma once
#include "zgemm.cuh"

namespace chase {

constexpr int FUSED_MAX_MEMBERS = 8;
constexpr int FUSED_QCAP = 8;        // owned tiles awaiting their peers' partials, per CTA

struct FusedArgs {
  int m;                                     // communicator members (2..8)
  int me;                                    // my index in the communicator
  double2* P[FUSED_MAX_MEMBERS];             // staging area of each member: m slots of ldP x n
  long long slot;                            // elements per slot
  double2* out[FUSED_MAX_MEMBERS];           // output buffer of each member (ld = g.ldo)
  unsigned* flags[FUSED_MAX_MEMBERS];        // arrival flags of each member: [tile * m + src]
  unsigned long long* done[FUSED_MAX_MEMBERS];  // delivery counter of each member
  long long ldP;
  unsigned ep;                               // epoch (unique per launch) written into flags
  unsigned long long done_target;            // wait for *done[me] >= done_target first
  int owner_beta;                            // owner adds beta * out(old) before broadcasting
  int* err;                                  // set on a spin timeout
  int plain;                                 // diagnostics: local epilogue, no protocol (m == 1)
  unsigned long long* tile_ctr;              // dynamic tile scheduler (monotonic, local)
  unsigned long long ctr_base;               // value of *tile_ctr at launch start (0: reset per launch)
  int tile_base;                             // flag index / owner offset of this launch's tiles
  int col_base;                              // staging-slot column offset of this launch's tiles
                                             //   (a step split into a wide-tile launch and a
                                             //   narrow-tile remainder launch keeps the two apart)
  int tiles;                                 // > 0: only the first `tiles` tiles of the raster (the
                                             //   rest is a split-K tail, fused_tail.cuh)
};

__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
constexpr long long FUSED_SPIN_CYCLES = 20000000000LL;   // ~10 s at 2 GHz

template <bool CONJ, int BN_ = ZG_BN>
__global__ void __launch_bounds__(ZG_THREADS, 1)
    zgemm_fused_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX,
                       const ZGemmArgs g, const FusedArgs f) {
  constexpr int WN_ = BN_ / ZG_WNW, NT_ = WN_ / 8;
  constexpr int XS_ = BN_ * 8 * 16, XB_ = XS_ * ZG_KS, SB_ = ZG_A_BYTES + XB_;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ZG_STAGES * SB_);
  uint64_t* empty = full + ZG_STAGES;
  __shared__ int s_abort;
  __shared__ int s_q[FUSED_QCAP];
  __shared__ int s_qh, s_qt, s_cmd;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = (g.N + BN_ - 1) / BN_, m_tiles = (g.M + ZG_BM - 1) / ZG_BM;
  const int T = f.tiles > 0 ? f.tiles : n_tiles * m_tiles;
  const int KT = (g.K + ZG_BK - 1) / ZG_BK;
  // dynamic tile scheduler: tiles come from a global counter into a small smem ring (tile -1 =
  // no more tiles).  k-tile issue index q maps to (seq, kt) = (q / KT, q % KT); the refill duty
  // rotates over the 8 MMA warps (as in zgemm.cuh), and a refill only sees the smem writes of
  // refills >= 2 iterations older (mbarrier ordering), so the tile of sequence position s is
  // grabbed two issue indices ahead, by the refill that issues q = s KT - 2.
  constexpr int RING = ZG_STAGES + 4;
  __shared__ int s_tile[RING];
  auto grab = [&]() -> int {
    const unsigned long long v = atomicAdd(f.tile_ctr, 1ull) - f.ctr_base;
    return v < (unsigned long long)T ? (int)v : -1;
  };
  auto tile_origin = [&](int t, int& m0, int& n0) {  // grouped rasterisation as in zgemm
    const int group = t / (ZG_GROUP_M * n_tiles);
    const int first_m = group * ZG_GROUP_M;
    const int gm = min(ZG_GROUP_M, m_tiles - first_m);
    const int within = t - group * ZG_GROUP_M * n_tiles;
    m0 = (first_m + within % gm) * ZG_BM;
    n0 = (within / gm) * BN_;
  };

  if (threadIdx.x == 0) {
    s_abort = 0;
    s_qh = s_qt = 0;
    // inputs of this step are complete once every owner of the previous step has delivered
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
    asm volatile("fence.proxy.async.global;" ::: "memory");   // peer stores -> TMA reads
    for (int s = 0; s < ZG_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ZG_CONSUMERS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (s_abort) return;

  // issue k-tile q into stage s (one lane); a stage past the last tile gets a plain arrive
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
    const int kt = q % KT;
    mbar_arrive_expect_tx(&full[s], SB_);
    uint8_t* sa = smem + s * SB_;
    uint8_t* sx = sa + ZG_A_BYTES;
#pragma unroll
    for (int u = 0; u < ZG_KS; ++u) {
      const int k0 = kt * ZG_BK + 8 * u;
      uint8_t* sau = sa + u * ZG_A_SLAB;
      if (CONJ) {
        tma_load_2d(sau, &tmA, 2 * (g.a_d0 + k0), g.a_d1 + m0, &full[s]);
      } else if (g.a3d) {
        tma_load_3d(sau, &tmA, 0, g.a_d1 + k0, (g.a_d0 + m0) / 8, &full[s]);
      } else {
#pragma unroll
        for (int b = 0; b < ZG_BM / 8; ++b)
          tma_load_2d(sau + b * 1024, &tmA, 2 * (g.a_d0 + m0 + 8 * b), g.a_d1 + k0, &full[s]);
      }
      tma_load_2d(sx + u * XS_, &tmX, 2 * (g.x_k0 + k0), g.x_n0 + n0, &full[s]);
    }
  };
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmX);
    for (int sq = 0; sq * KT < 2; ++sq) s_tile[sq % RING] = grab();   // tiles with q_grab < 0
    for (int gs = 0; gs < ZG_STAGES; ++gs) issue(gs, gs);
  }

  const int wm = warp & 3, wn = warp >> 2;
  const int gq = lane >> 2, tq = lane & 3;
  double acc_re[2][NT_][4], acc_im[2][NT_][4];
  auto zero_acc = [&]() {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < NT_; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc_re[i][j][r] = acc_im[i][j][r] = 0.0;
  };
  zero_acc();

  constexpr int SUBS = 2 * ZG_KS;
  struct Frag {
    double2 a[2][2], b[NT_];
  };
  auto load = [&](Frag& fr, int gs, int kt, int sub) {
    const int u = sub >> 1, h = sub & 1;
    const int k = 2 * tq + h;
    const uint8_t* sa = smem + (gs % ZG_STAGES) * SB_ + u * ZG_A_SLAB;
    const uint8_t* sx = smem + (gs % ZG_STAGES) * SB_ + ZG_A_BYTES + u * XS_;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int m = wm * 32 + mt * 16 + r * 8 + gq;
        const int off = CONJ ? m * 128 + ((k ^ gq) << 4) : (m >> 3) * 1024 + k * 128 + ((gq ^ k) << 4);
        fr.a[mt][r] = *reinterpret_cast<const double2*>(sa + off);
      }
#pragma unroll
    for (int nt = 0; nt < NT_; ++nt) {
      const int n = wn * WN_ + nt * 8 + gq;
      fr.b[nt] = *reinterpret_cast<const double2*>(sx + n * 128 + ((k ^ gq) << 4));
    }
    if (kt * ZG_BK + 8 * u + k >= g.K) {
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) fr.a[mt][0] = fr.a[mt][1] = make_double2(0.0, 0.0);
#pragma unroll
      for (int nt = 0; nt < NT_; ++nt) fr.b[nt] = make_double2(0.0, 0.0);
    }
  };
  auto mma = [&](const Frag& fr) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT_; ++nt) {
        dmma_16x8x4(acc_re[mt][nt], fr.a[mt][0].x, fr.a[mt][1].x, fr.b[nt].x);
        dmma_16x8x4(acc_im[mt][nt], fr.a[mt][0].x, fr.a[mt][1].x, fr.b[nt].y);
      }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT_; ++nt) {
        const double bre = CONJ ? fr.b[nt].y : -fr.b[nt].y;
        const double bim = CONJ ? -fr.b[nt].x : fr.b[nt].x;
        dmma_16x8x4(acc_re[mt][nt], fr.a[mt][0].y, fr.a[mt][1].y, bre);
        dmma_16x8x4(acc_im[mt][nt], fr.a[mt][0].y, fr.a[mt][1].y, bim);
      }
  };

  // owner side: fixed-order sum of the m partial tiles of t (local slots), + beta V_{s-2},
  // broadcast into every member's output, delivery counters bumped
  auto reduce = [&](int t) {
    int m0, n0;
    tile_origin(t, m0, n0);
    // coalesced pass over the tile (column-major 128 x 64), partials read from local slots;
    // 8 elements per thread per batch so the loads of a batch are all in flight together
    const double2* __restrict__ mine = f.P[f.me];
    constexpr int PER = ZG_BM * BN_ / ZG_THREADS;     // 32 elements per thread
    constexpr int BATCH = 8;
#pragma unroll 1
    for (int b0 = 0; b0 < PER; b0 += BATCH) {
      double2 sum[BATCH];
      long long io[BATCH];
      bool ok[BATCH];
#pragma unroll
      for (int i = 0; i < BATCH; ++i) {
        const int e = threadIdx.x + (b0 + i) * ZG_THREADS;
        const int row = m0 + (e % ZG_BM), col = n0 + (e / ZG_BM);
        ok[i] = row < g.M && col < g.N;
        const long long ip = (long long)row + (long long)(f.col_base + col) * f.ldP;
        io[i] = (long long)row + (long long)col * g.ldo;
        sum[i] = ok[i] ? mine[ip] : make_double2(0.0, 0.0);
        for (int src = 1; src < f.m; ++src) {
          const double2 v = ok[i] ? mine[(long long)src * f.slot + ip] : make_double2(0.0, 0.0);
          sum[i].x += v.x;
          sum[i].y += v.y;
        }
        if (f.owner_beta && ok[i]) {
          const double2 old = f.out[f.me][io[i]];
          sum[i].x += g.beta * old.x;
          sum[i].y += g.beta * old.y;
        }
      }
#pragma unroll
      for (int i = 0; i < BATCH; ++i)
        if (ok[i])
          for (int dst = 0; dst < f.m; ++dst) f.out[dst][io[i]] = sum[i];
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

  // epilogue of tile t: publish the partial, and reduce + broadcast it if this member owns t
  auto epilogue = [&](int t) {
    int m0, n0;
    tile_origin(t, m0, n0);
    if (f.plain) {
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
              if (row >= g.band_lo && row < g.band_hi) {
                const double2 x = g.xin[(long long)(row + g.band_shift) + (long long)col * g.ldx];
                vr -= g.c * x.x;
                vi -= g.c * x.y;
              }
              vr *= g.alpha;
              vi *= g.alpha;
              double2* o = f.out[f.me] + (long long)row + (long long)col * g.ldo;
              if (f.owner_beta) {
                const double2 old = *o;
                vr += g.beta * old.x;
                vi += g.beta * old.y;
              }
              *o = make_double2(vr, vi);
            }
          }
      if (threadIdx.x == 0) atomicAdd(f.done[f.me], 1ull);
      return;
    }
    // owner = t mod m: consecutive tiles (those in flight together) go to different members
    const int owner = (f.tile_base + t) % f.m;
    double2* slot = f.P[owner] + (long long)f.me * f.slot;        // my slot at the owner
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
            slot[(long long)row + (long long)(f.col_base + col) * f.ldP] = make_double2(vr * g.alpha, vi * g.alpha);
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
  int seq = 0, kt = 0, gs = 0;
  for (;;) {
    const int s = gs % ZG_STAGES;
    int next_tile = tile;
#pragma unroll
    for (int sub = 0; sub < SUBS; ++sub) {
      if (sub + 1 < SUBS) {
        load(nxt, gs, kt, sub + 1);
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        mbar_wait_dbg(&full[(gs + 1) % ZG_STAGES], ((gs + 1) / ZG_STAGES) & 1, 2, gs);
        if (kt + 1 < KT) {
          load(nxt, gs + 1, kt + 1, 0);
        } else {
          next_tile = s_tile[(seq + 1) % RING];
          if (next_tile >= 0) load(nxt, gs + 1, 0, 0);
        }
      }
      mma(cur);
      cur = nxt;
    }
    // refill the stage released one iteration ago; the duty rotates over the warps
    if (lane == 0 && warp == (gs & (ZG_CONSUMERS - 1)) && gs >= 1) {
      const int sp = (gs - 1) % ZG_STAGES;
      mbar_wait_dbg(&empty[sp], ((gs - 1) / ZG_STAGES) & 1, 3, gs);
      issue(gs - 1 + ZG_STAGES, sp);
    }
    ++gs;
    if (++kt == KT) {
      epilogue(tile);
      zero_acc();
      if (s_abort) {              // a peer never arrived: give up (the host reports CHASE_ECUDA)
        // every refill up to iteration gs - 1 is done (the epilogue synchronised the CTA): let the
        // loads of issue indices gs .. gs + STAGES - 2 land before the CTA exits
        if (threadIdx.x == 0)
          for (int r = gs; r < gs + ZG_STAGES - 1; ++r) mbar_wait(&full[r % ZG_STAGES], (r / ZG_STAGES) & 1);
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

// Waits (one thread) until *done >= target: the last step's tiles are all delivered before the
// result is copied out of the symmetric buffer.
__global__ void fused_wait_kernel(const unsigned long long* done, unsigned long long target, int* err) {
  const long long t0 = clock64();
  while (ld_acquire_sys_u64(done) < target) {
    __nanosleep(256);
    if (clock64() - t0 > FUSED_SPIN_CYCLES) {
      atomicExch(err, 1);
      return;
    }
  }
}

}  // namespace chase
