// fused_tail.cuh -- wave-quantisation tail of the fused filter step (zgemm_fused.cuh).
//
// The persistent fused kernel hands out a step's T output tiles one by one; when T is not a
// multiple of its grid G the last round leaves G - T mod G CTAs idle for a whole tile time (R5 on
// 2 x 4: K = 100000, one real tile ~13 ms).  As for the plain GEMM (gemm_tail.cuh) the host then
// runs the fused kernel on the first T_main tiles only and the last T_tail tiles as S split-K
// copies (zgemm/dgemm SPLIT variant, tile-local partials in the local tail workspace).  Their
// reduction over the communicator is done here through peer memory, without an owner, in the
// push style of the fused kernel (remote stores, local reads):
//   1. publish (one CTA per tail tile): the S partials summed in fixed order, the band term and
//      alpha applied -- this member's partial of the tile -- stored into sub-slot [me] of the tail
//      slot of EVERY member (NVLink stores);
//   2. sync (one thread): release this member's flag in every member's flag array, then wait
//      until the flags of all m members carry this launch's epoch;
//   3. reduce (one CTA per tail tile): every member sums the m partials in its LOCAL sub-slots in
//      fixed member order, adds beta * V_{s-2} (replicated) and writes its own output -- identical
//      bits on every member, no broadcast, no delivery counter.
// Only the sync kernel spins (one thread, so it can share an SM with a persistent fused CTA of a
// peer on the same device: virtual grids).  Tail slots alternate per step parity: a peer can
// publish the next same-parity step before this member has read the current one (other slot),
// but not the one after (its sync needs this member's flag of the next step, released after this
// member's reduce of the current one in stream order).
#pragma once
#include "gemm_tail.cuh"
#include "zgemm_fused.cuh"

namespace chase {

constexpr int FUSED_TAIL_SLOTS = 4;          // tail slots (and flag arrays): 2 per step parity
constexpr int FUSED_TAIL_TILES = 320;        // tail tiles held per sub-slot (128 KB places)

struct FusedTailArgs {
  int m, me;                                 // communicator members, my index
  int S, tail_tiles, tile_offset, slot_off;  // split copies; tail tiles; first tail tile; slot offset
  int M, N;
  long long ldo, ldx;
  double alpha, beta, c;
  int owner_beta, band_lo, band_hi, band_shift;
  const int* band_map;
  void* tp[FUSED_MAX_MEMBERS];               // tail slot of each member: m sub-slots [src] of
  long long sub;                             //   `sub` elements (tile-local partial tiles)
  unsigned* tflag[FUSED_MAX_MEMBERS];        // tail flags of each member, [src]
  unsigned ep;
  int* err;
};

// every tail tile takes one 128 KB place in a sub-slot whatever its shape (wide and narrow tiles
// of one step share the slot; slot_off counts places)
template <typename T> constexpr long long FT_TILE_ELEMS = 131072 / sizeof(T);

template <typename T> __device__ __forceinline__ T tl_zero();
template <> __device__ __forceinline__ double tl_zero<double>() { return 0.0; }
template <> __device__ __forceinline__ double2 tl_zero<double2>() { return make_double2(0.0, 0.0); }

template <int BM, int BN, int GROUP_M>
__device__ __forceinline__ void tl_origin(int t, int M, int N, int& m0, int& n0) {
  const int n_tiles = (N + BN - 1) / BN, m_tiles = (M + BM - 1) / BM;
  const int group = t / (GROUP_M * n_tiles);
  const int first_m = group * GROUP_M;
  const int gm = min(GROUP_M, m_tiles - first_m);
  const int within = t - group * GROUP_M * n_tiles;
  m0 = (first_m + within % gm) * BM;
  n0 = (within / gm) * BN;
}

template <typename T, int BM, int BN, int GROUP_M>
__global__ void __launch_bounds__(256)
    fused_tail_publish_kernel(const T* __restrict__ part, const T* xin, const FusedTailArgs a) {
  static_assert(BM * BN <= FT_TILE_ELEMS<T>, "tail tile larger than its slot place");
  const int j = blockIdx.x;
  int m0, n0;
  tl_origin<BM, BN, GROUP_M>(a.tile_offset + j, a.M, a.N, m0, n0);
  const long long off = (long long)a.me * a.sub + (long long)(a.slot_off + j) * FT_TILE_ELEMS<T>;
  for (int e = threadIdx.x; e < BM * BN; e += blockDim.x) {
    const int row = m0 + (e % BM), col = n0 + (e / BM);
    T acc = tl_zero<T>();
    if (row < a.M && col < a.N) {
      acc = part[(long long)j * (BM * BN) + e];
      for (int s = 1; s < a.S; ++s) acc = tl_add(acc, part[((long long)s * a.tail_tiles + j) * (BM * BN) + e]);
      const int bsrc = a.band_map != nullptr ? a.band_map[row]
                       : (row >= a.band_lo && row < a.band_hi ? row + a.band_shift : -1);
      if (bsrc >= 0) acc = tl_axpy(acc, a.c, xin[(long long)bsrc + (long long)col * a.ldx]);
      acc = tl_scale(acc, a.alpha);
    }
    for (int dst = 0; dst < a.m; ++dst) static_cast<T*>(a.tp[dst])[off + e] = acc;
  }
}

__global__ void fused_tail_sync_kernel(const FusedTailArgs a) {
  __threadfence_system();                                   // the publish kernel's stores
  for (int dst = 0; dst < a.m; ++dst) st_release_sys_u32(a.tflag[dst] + a.me, a.ep);
  const long long t0 = clock64();
  for (int src = 0; src < a.m; ++src) {
    while (ld_acquire_sys_u32(a.tflag[a.me] + src) != a.ep) {
      __nanosleep(128);
      if (clock64() - t0 > FUSED_SPIN_CYCLES) {
        printf("[chase fused tail] member %d: partial of member %d missing (ep %u)\n", a.me, src, a.ep);
        atomicExch(a.err, 1);
        return;
      }
    }
  }
  __threadfence_system();
}

template <typename T, int BM, int BN, int GROUP_M>
__global__ void __launch_bounds__(256) fused_tail_reduce_kernel(T* out, const FusedTailArgs a) {
  const int j = blockIdx.x;
  int m0, n0;
  tl_origin<BM, BN, GROUP_M>(a.tile_offset + j, a.M, a.N, m0, n0);
  const T* mine = static_cast<const T*>(a.tp[a.me]) + (long long)(a.slot_off + j) * FT_TILE_ELEMS<T>;
  for (int e = threadIdx.x; e < BM * BN; e += blockDim.x) {
    const int row = m0 + (e % BM), col = n0 + (e / BM);
    if (row >= a.M || col >= a.N) continue;
    T acc = mine[e];
    for (int src = 1; src < a.m; ++src) acc = tl_add(acc, mine[(long long)src * a.sub + e]);
    T* o = out + (long long)row + (long long)col * a.ldo;
    if (a.owner_beta) acc = tl_fma(acc, a.beta, *o);
    *o = acc;
  }
}

}  // namespace chase
