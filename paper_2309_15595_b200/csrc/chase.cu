// chase.cu -- host side of libchase.so: handle, argument validation, the filter step driver,
// the 1D-CAQR driver (Alg.4) and the C-ABI declared in include/chase.h.
//
// Every step of the hot path runs in this library's kernels (zgemm.cuh, qr_kernels.cuh) and
// NCCL collectives on the handle's stream; there is no CPU fallback.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: phase ranges for nsys / ncu --nvtx

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "chase.h"
#include "dgemm.cuh"
#include "eig.cuh"
#include "hhqr.cuh"
#include "gemm_tail.cuh"
#include "qr_kernels.cuh"
#include "tridiag.cuh"
#include "zgemm.cuh"
#include "zgemm_fused.cuh"
#include "dgemm_fused.cuh"
#include "fused_tail.cuh"

using namespace chase;

// ==================================================================== utilities
#define CUDA_TRY(x)                                                                   \
  do {                                                                                \
    cudaError_t err__ = (x);                                                          \
    if (err__ != cudaSuccess) {                                                       \
      fprintf(stderr, "[chase] CUDA error %s at %s:%d\n", cudaGetErrorString(err__), \
              __FILE__, __LINE__);                                                    \
      return CHASE_ECUDA;                                                             \
    }                                                                                 \
  } while (0)
#define NCCL_TRY(x)                                                                   \
  do {                                                                                \
    ncclResult_t r__ = (x);                                                           \
    if (r__ != ncclSuccess) {                                                         \
      fprintf(stderr, "[chase] NCCL error %s at %s:%d\n", ncclGetErrorString(r__),    \
              __FILE__, __LINE__);                                                    \
      return CHASE_ENCCL;                                                             \
    }                                                                                 \
  } while (0)
#define STATUS_TRY(x)                 \
  do {                                \
    chase_status_t st__ = (x);        \
    if (st__ != CHASE_OK) return st__; \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2D FP64 tensor map over a column-major matrix of `rows` x `cols` elements of `esize` bytes
// (16 = complex, 8 = real), leading dimension ld (elements), box = box_rows x box_cols elements,
// 128-byte swizzle (box_rows * esize must be 128).
static chase_status_t make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols,
                               int64_t ld, int esize, int box_rows, int box_cols) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return CHASE_ECUDA;
  const int per = esize / 8;
  cuuint64_t dims[2] = {(cuuint64_t)(rows * per), (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * esize)};
  cuuint32_t box[2] = {(cuuint32_t)(box_rows * per), (cuuint32_t)box_cols};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "[chase] cuTensorMapEncodeTiled failed (%d): rows %lld cols %lld ld %lld\n",
            (int)r, (long long)rows, (long long)cols, (long long)ld);
    return CHASE_ECUDA;
  }
  return CHASE_OK;
}

// Block-cyclic distribution with block size nb over P grid rows/columns: grid
// row k owns global rows g with (g / nb) mod P == k, in increasing order.
static void cyclic_indices(int64_t N, int P, int k, int64_t nb, std::vector<int64_t>* idx) {
  idx->clear();
  for (int64_t b = k; b * nb < N; b += P)
    for (int64_t g = b * nb; g < std::min(N, (b + 1) * nb); ++g) idx->push_back(g);
}

static void block_part(int64_t N, int P, int k, int64_t* size, int64_t* start) {
  const int64_t b = N / P, rem = N % P;
  *size = b + (k < rem ? 1 : 0);
  *start = k * b + (k < rem ? k : rem);
}

// ==================================================================== handle
enum { CAT_HEMM_ODD = 0, CAT_HEMM_EVEN, CAT_ALLREDUCE, CAT_GRAM, CAT_POTRF, CAT_TRSM, CAT_OTHER,
       CAT_HHQR, CAT_N };

struct chase_handle_s {
  chase_dtype_t dt;
  int64_t N, n_max;
  int p, q, myrow, mycol;
  int64_t n_r, n_c, r0, c0;       // r0 = c0 = -1 for the block-cyclic distribution
  int64_t nb = 0;                 // block-cyclic block size (0 = block distribution)
  int64_t voff = 0;               // first "virtual" row of this rank in the column communicator
                                  //   (rank 0's rows, rank 1's, ...): the HHQR row order
  int qr_mode = 0;                // 0: Alg.4 dispatch; 1: Householder QR always (Table 3)
  std::vector<int64_t> rows_g, cols_g;   // global indices of the local rows / columns
  int* d_band_odd = nullptr;      // block-cyclic: B-layout row -> C-layout row of the diagonal
  int* d_band_even = nullptr;     //   C-layout row -> B-layout row of the diagonal (or -1)
  int* d_b2_src = nullptr;        // residual B2 redistribution: per owning grid row, the source
  int* d_b2_dst = nullptr;        //   local rows (on the owner) and the B2 rows they fill
  std::vector<int64_t> b2_seg;    //   segment offsets, p + 1 entries
  int device;
  cudaStream_t stream;
  ncclComm_t world = nullptr, rcomm = nullptr, ccomm = nullptr;
  // workspace
  void* ws = nullptr;
  size_t ws_bytes = 0;
  void* Bws = nullptr;      // n_c x n_max (B-layout block)
  void* Gws = nullptr;      // n_max x n_max (Gram / R)
  void* Wws = nullptr;      // n_r x n_max (TRSM output)
  void* Rinv = nullptr;     // 64 x n_max (inverted diagonal blocks of R)
  char* Rfws = nullptr;     // R^{-1} n_max x n_max, then the recursive-doubling temp
  void* B2ws = nullptr;     // n_c x n_max (C redistributed into B-layout, Alg.2 l.23)
  char* eigws = nullptr;    // Jacobi eigensolver region (see eig_bytes)
  char* c2ws = nullptr;     // solver: C2
  char* lanws = nullptr;    // solver: Lanczos basis
  char* hhws = nullptr;     // Householder QR fallback (see hh_layout)
  char* tailws = nullptr;   // split-K tail partial tiles (gemm_tail.cuh)
  double* d_ritz = nullptr;
  double* d_nrm = nullptr;
  int* d_info = nullptr;
  double* d_shift = nullptr;
  int* h_info = nullptr;    // pinned
  double* h_shift = nullptr;   // pinned: the shift of the last shifted CholeskyQR pass
  double last_shift = 0.0;
  // virtual grid (chase_create_virtual): every rank of the grid lives in this process on one
  // device, no NCCL communicators; reductions only through the fused peer-memory path
  bool virt = false;
  // fused compute+collective filter (symmetric peer memory); see zgemm_fused.cuh
  bool fused = false;
  int fused_mode = 0;             // 1: single-member steps also run the fused kernel (self)
  int sm_budget = 0;              // > 0: persistent fused grids use at most this many CTAs
  bool fused_broken = false;      // a peer wait timed out: chase_set_fused_workspace again
  char* fz_base[FUSED_MAX_MEMBERS * FUSED_MAX_MEMBERS] = {nullptr};   // per world rank
  int world_size = 1;
  unsigned fused_ep = 0;
  unsigned long long fused_delivered = 0;
  unsigned fused_tail_k[2] = {0, 0};  // fused odd / even steps so far: tail slot rotation
  int* d_err = nullptr;
  int num_sms = 148;
  // bookkeeping of the last filter call
  std::vector<chase_step_record_t> record;
  int64_t last_matvecs = 0;
  // profiling
  bool profiling = false;
  struct Ev {
    int cat;
    cudaEvent_t a, b;
  };
  std::vector<Ev> evs;
  std::vector<cudaEvent_t> pool;
  int64_t launches[CAT_N] = {0};

  cudaEvent_t ev_get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

// NVTX range around a host scope (an API call or a phase); free when no tool is attached
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};
static const char* const kCatName[CAT_N] = {"hemm_odd (A^H C -> B)", "hemm_even (A B -> C)", "allreduce",
                                            "gram", "potrf", "trsm", "other", "hhqr"};

struct ProfScope {
  chase_handle_s* h;
  int cat;
  cudaEvent_t a = nullptr;
  Nvtx range;
  ProfScope(chase_handle_s* h_, int c, int nlaunch) : h(h_), cat(c), range(kCatName[c]) {
    h->launches[c] += nlaunch;
    if (h->profiling) {
      a = h->ev_get();
      cudaEventRecord(a, h->stream);
    }
  }
  ~ProfScope() {
    if (h->profiling) {
      cudaEvent_t b = h->ev_get();
      cudaEventRecord(b, h->stream);
      h->evs.push_back({cat, a, b});
    }
  }
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
// Leading dimension of library-owned buffers: even, so every column starts 16-byte aligned
// (TMA requires 16-byte global strides; matters for real double).
static int64_t pad_ld(int64_t rows) { return (rows + 1) & ~(int64_t)1; }

static size_t esize_of(chase_dtype_t dt) { return dt == CHASE_C128 ? 16 : 8; }

constexpr int TAIL_TILES_MAX = 320;   // split-K tail: tiles x copies held (128 KB each)
struct WsLayout {
  size_t b, g, w, rinv, rf, b2, ritz, nrm, maps, eig, c2, lan, hh, tail, info, s, total;
};
constexpr int LANCZOS_K = 25;       // Lanczos steps per run (bounds, Alg.1 l.2)
constexpr int LANCZOS_RUNS = 4;     // independent runs pooled for the DoS estimate
// Jacobi eigensolver buffers (Rayleigh-Ritz): A ping-pong, Y ping-pong, U_bd (np x np complex
// each, np = n_max rounded up to 64) + eigenvalues, order, permutation tables, partial sums.
static int64_t eig_np(int64_t n) { return (n + JAC_PW - 1) / JAC_PW * JAC_PW; }
static size_t eig_bytes(int64_t n_max) {
  const int64_t np = eig_np(n_max), L = np / 32;
  return 5 * align256((size_t)np * np * 16) + align256(np * sizeof(double)) +
         align256(np * sizeof(int)) + align256((size_t)(L + 1) * L * sizeof(int)) +
         align256(2 * JAC_RED_BLOCKS * sizeof(double) + 2 * sizeof(double)) +
         align256((size_t)(2 * 128 * np + 2 * 128 * 128) * 16);   // tridiagonal back-transform
}
// Householder QR scratch: panel reflectors Vp (n_r x 128), the compact-WY factors T of every
// panel (128 x n_max), two 128 x n_max products, S = Vp^H Vp, tau, beta, CTA partials, split-K
// partial products, reduced scalars and the arrival counters.
struct HhLayout {
  size_t vp, t, wb, wb2, s, tau, beta, part, psplit, red_n, red_w, ctr, total;
  int64_t split_cols;     // columns of HH_NB-row split-K partials the psplit buffer holds
};
static HhLayout hh_layout(const chase_handle_s* h) {
  const size_t es = esize_of(h->dt);
  HhLayout L;
  size_t off = 0;
  L.vp = off;   off += align256((size_t)pad_ld(h->n_r) * HH_NB * es);
  L.t = off;    off += align256((size_t)HH_NB * (h->n_max + HH_NB) * es);
  L.wb = off;   off += align256((size_t)HH_NB * h->n_max * es);
  L.wb2 = off;  off += align256((size_t)HH_NB * h->n_max * es);
  L.s = off;    off += align256((size_t)HH_NB * HH_NB * es);
  L.tau = off;  off += align256((size_t)h->n_max * es);
  L.beta = off; off += align256((size_t)h->n_max * sizeof(double));
  L.part = off; off += align256((size_t)(HH_NCH + 1) * HH_GRID_MAX * HH_CH * 16);
  L.split_cols = std::max<int64_t>(h->n_max, std::min<int64_t>(2 * 148 * 64, 64 * h->n_max));
  L.psplit = off; off += align256((size_t)HH_NB * L.split_cols * es);
  L.red_n = off; off += 256;
  L.red_w = off; off += align256((size_t)HH_NB * 16);
  L.ctr = off;  off += 256;
  L.total = off;
  return L;
}

// B-layout block (n_c x n_max) | Gram/R (n_max x n_max) | TRSM output W (n_r x n_max)
// | inverted diagonal blocks of R (64 x n_max) | info | shift
static WsLayout ws_layout(const chase_handle_s* h) {
  const size_t es = esize_of(h->dt);
  WsLayout L;
  size_t off = 0;
  L.b = off;
  off += align256((size_t)pad_ld(h->n_c) * h->n_max * es);
  L.g = off;
  off += align256((size_t)pad_ld(h->n_max) * h->n_max * es);
  L.w = off;                                            // also the residual Bcast staging area
  off += align256((size_t)(std::max(h->n_r, h->n_c) + 2) * h->n_max * es);
  L.rinv = off;
  off += align256((size_t)TRTRI_NB * (h->n_max + TRTRI_NB) * es);
  L.rf = off;                                           // R^{-1} (n_max^2) + doubling temp
  off += 2 * align256((size_t)pad_ld(h->n_max) * h->n_max * es);
  L.b2 = off;                                           // residual: C redistributed to B-layout
  off += align256((size_t)pad_ld(h->n_c) * h->n_max * es);
  L.ritz = off;
  off += align256((size_t)h->n_max * sizeof(double));
  L.nrm = off;
  off += align256((size_t)h->n_max * sizeof(double));
  L.maps = off;                                         // block-cyclic index maps (int32)
  off += align256((size_t)(h->n_r + 3 * h->n_c) * sizeof(int));
  L.eig = off;                                          // Rayleigh-Ritz eigensolver
  off += eig_bytes(h->n_max);
  L.c2 = off;                                           // solver: C2 (Alg.2 buffers C2 / B2)
  off += align256((size_t)pad_ld(h->n_r) * h->n_max * es);
  L.lan = off;                                          // solver: Lanczos basis + scalars
  off += align256((size_t)pad_ld(h->n_r) * (LANCZOS_K + 2) * es) + 4096;
  L.hh = off;                                           // Householder QR fallback
  off += hh_layout(h).total;
  L.tail = off;                                         // split-K tail partial tiles
  off += align256((size_t)TAIL_TILES_MAX * 128 * 128 * 8);
  L.info = off;
  off += 256;
  L.s = off;
  off += 256;
  L.total = off;
  return L;
}


// ==================================================================== GEMM launchers
static bool g_disable_a3d = getenv("CHASE_DISABLE_A3D") != nullptr;   // A/B switch for tuning

// (dynamic shared memory sizes of every variant are set once by preload_kernels)
static chase_status_t launch_zgemm(chase_handle_s* h, bool conj, const CUtensorMap& tA,
                                   const CUtensorMap& tX, const ZGemmArgs& a, int grid_tiles = 0,
                                   bool narrow = false, int nbatch = 1, bool ext = false) {
  if (a.M <= 0 || a.N <= 0) return CHASE_OK;
  const bool split = a.k_split > 1;
  const int BN = narrow ? ZG_BN_NARROW : ZG_BN;
  const int tiles = a.tail_tiles > 0 ? a.tail_tiles
                    : grid_tiles > 0 ? grid_tiles
                                     : ((a.N + BN - 1) / BN) * ((a.M + ZG_BM - 1) / ZG_BM);
  dim3 grid(tiles * (split ? a.k_split : 1), std::max(1, nbatch));
  auto go = [&](auto kern, int smem) -> chase_status_t {
    kern<<<grid, ZG_THREADS, smem, h->stream>>>(tA, tX, a);
    CUDA_TRY(cudaGetLastError());
    return CHASE_OK;
  };
  constexpr int S = ZG_SMEM_BYTES, SN = zg_smem_bytes(ZG_BN_NARROW);
  if (ext) {                                     // tri_k / batched (TRSM, TRTRI): NoTrans, plain
    if (conj || split || narrow) return CHASE_EINVAL;
    return go(zgemm_kernel<false, false, ZG_BN, true>, S);
  }
  if (narrow) {
    if (conj) return split ? go(zgemm_kernel<true, true, ZG_BN_NARROW>, SN) : go(zgemm_kernel<true, false, ZG_BN_NARROW>, SN);
    return split ? go(zgemm_kernel<false, true, ZG_BN_NARROW>, SN) : go(zgemm_kernel<false, false, ZG_BN_NARROW>, SN);
  }
  if (conj) return split ? go(zgemm_kernel<true, true>, S) : go(zgemm_kernel<true>, S);
  return split ? go(zgemm_kernel<false, true>, S) : go(zgemm_kernel<false>, S);
}

static chase_status_t launch_zgemm_fused(chase_handle_s* h, bool conj, const CUtensorMap& tA,
                                         const CUtensorMap& tX, const struct GemmReq& r,
                                         const FusedArgs& f, int T, bool narrow);

static chase_status_t launch_dgemm(chase_handle_s* h, bool trans, const CUtensorMap& tA,
                                   const CUtensorMap& tX, const DGemmArgs& a, int grid_tiles = 0,
                                   bool narrow = false, int nbatch = 1, bool ext = false) {
  if (a.M <= 0 || a.N <= 0) return CHASE_OK;
  const bool split = a.k_split > 1;
  const int BN = narrow ? DG_BN_NARROW : DG_BN;
  const int tiles = a.tail_tiles > 0 ? a.tail_tiles
                    : grid_tiles > 0 ? grid_tiles
                                     : ((a.N + BN - 1) / BN) * ((a.M + DG_BM - 1) / DG_BM);
  dim3 grid(tiles * (split ? a.k_split : 1), std::max(1, nbatch));
  auto go = [&](auto kern, int smem) -> chase_status_t {
    kern<<<grid, DG_THREADS, smem, h->stream>>>(tA, tX, a);
    CUDA_TRY(cudaGetLastError());
    return CHASE_OK;
  };
  constexpr int S = dg_smem_bytes(DG_BN), SN = dg_smem_bytes(DG_BN_NARROW);
  if (ext) {                                     // tri_k / batched (TRSM, TRTRI): NoTrans, plain
    if (trans || split || narrow) return CHASE_EINVAL;
    return go(dgemm_kernel<false, false, DG_BN, true>, S);
  }
  if (narrow) {
    if (trans) return split ? go(dgemm_kernel<true, true, DG_BN_NARROW>, SN) : go(dgemm_kernel<true, false, DG_BN_NARROW>, SN);
    return split ? go(dgemm_kernel<false, true, DG_BN_NARROW>, SN) : go(dgemm_kernel<false, false, DG_BN_NARROW>, SN);
  }
  if (trans) return split ? go(dgemm_kernel<true, true>, S) : go(dgemm_kernel<true>, S);
  return split ? go(dgemm_kernel<false, true>, S) : go(dgemm_kernel<false>, S);
}

// One generic GEMM request, dispatched on the handle's dtype.  Pointers are element pointers
// of the handle's dtype; offsets are in elements.
struct GemmReq {
  bool conj;                 // opA = A^H (A^T for real)
  const CUtensorMap* tA;
  const CUtensorMap* tX;
  int M, N, K, a_d0, a_d1, x_k0, x_n0;
  void* out;
  int64_t ldo;
  const void* xin;
  int64_t ldx;
  double alpha, beta, c;
  int use_beta, band_lo, band_hi, band_shift, upper_only;
  const int* abort_flag;
  const int* band_map;       // block-cyclic band (device), replaces band_lo/hi/shift
  int diag_k;                // block-diagonal k ranges (eigensolver updates), complex only
  int a3d;                   // NoTrans: tA is the 3D single-box view (a_d0 multiple of a piece)
  const double* col_shift;   // residual epilogue (Alg.2 l.25): out -= col_shift[n] y2(m, n)
  const void* y2;
  int64_t ldy2;
  int k_split;               // split-K copies (> 1: partial products at out + s * split_ld)
  int64_t split_ld;
  int tail_tiles, tile_offset;  // split-K tail launch (see gemm_tail.cuh)
  int grid_tiles;            // > 0: launch only the first grid_tiles tiles of the raster
  int narrow;                // the narrow-tile variant (BN = ZG/DG_BN_NARROW); tX has its box
  const CUtensorMap* tX_narrow;   // run_gemm_tail: X map with the narrow box -> remainder split
  int tri_k;                 // X upper triangular: per-tile K = min(K, n0 + BN) (TRSM by R^{-1})
  int nbatch;                // > 1: batched launch (gridDim.y), strides bat_a / bat_x / bat_out
  int bat_a, bat_x;
  int64_t bat_out;
};

static chase_status_t run_gemm(chase_handle_s* h, const GemmReq& r) {
  if (h->dt == CHASE_C128) {
    ZGemmArgs a{};
    a.tri_k = r.tri_k;
    a.bat_a = r.bat_a; a.bat_x = r.bat_x; a.bat_out = r.bat_out;
    a.M = r.M; a.N = r.N; a.K = r.K;
    a.a_d0 = r.a_d0; a.a_d1 = r.a_d1; a.x_k0 = r.x_k0; a.x_n0 = r.x_n0;
    a.out = static_cast<double2*>(r.out); a.ldo = r.ldo;
    a.xin = static_cast<const double2*>(r.xin); a.ldx = r.ldx;
    a.alpha = r.alpha; a.beta = r.beta; a.c = r.c;
    a.use_beta = r.use_beta; a.band_lo = r.band_lo; a.band_hi = r.band_hi;
    a.band_shift = r.band_shift; a.upper_only = r.upper_only; a.abort_flag = r.abort_flag;
    a.band_map = r.band_map;
    a.diag_k = r.diag_k;
    a.a3d = r.a3d;
    a.col_shift = r.col_shift; a.y2 = static_cast<const double2*>(r.y2); a.ldy2 = r.ldy2;
    a.k_split = r.k_split; a.split_ld = r.split_ld;
    a.tail_tiles = r.tail_tiles; a.tile_offset = r.tile_offset;
    return launch_zgemm(h, r.conj, *r.tA, *r.tX, a, r.grid_tiles, r.narrow != 0, r.nbatch,
                        r.tri_k != 0 || r.nbatch > 1);
  }
  DGemmArgs a{};
  a.tri_k = r.tri_k;
  a.bat_a = r.bat_a; a.bat_x = r.bat_x; a.bat_out = r.bat_out;
  a.M = r.M; a.N = r.N; a.K = r.K;
  a.a_d0 = r.a_d0; a.a_d1 = r.a_d1; a.x_k0 = r.x_k0; a.x_n0 = r.x_n0;
  a.out = static_cast<double*>(r.out); a.ldo = r.ldo;
  a.xin = static_cast<const double*>(r.xin); a.ldx = r.ldx;
  a.alpha = r.alpha; a.beta = r.beta; a.c = r.c;
  a.use_beta = r.use_beta; a.band_lo = r.band_lo; a.band_hi = r.band_hi;
  a.band_shift = r.band_shift; a.upper_only = r.upper_only; a.abort_flag = r.abort_flag;
  a.band_map = r.band_map;
  a.diag_k = r.diag_k;
  a.a3d = r.a3d;
  a.col_shift = r.col_shift; a.y2 = static_cast<const double*>(r.y2); a.ldy2 = r.ldy2;
  a.k_split = r.k_split; a.split_ld = r.split_ld;
  a.tail_tiles = r.tail_tiles; a.tile_offset = r.tile_offset;
  return launch_dgemm(h, r.conj, *r.tA, *r.tX, a, r.grid_tiles, r.narrow != 0, r.nbatch,
                      r.tri_k != 0 || r.nbatch > 1);
}

static chase_status_t launch_dgemm_fused(chase_handle_s* h, bool trans, const CUtensorMap& tA,
                                         const CUtensorMap& tX, const GemmReq& r,
                                         const FusedArgs& f, int T, bool narrow) {
  DGemmArgs a{};
  a.M = r.M; a.N = r.N; a.K = r.K;
  a.a_d0 = r.a_d0; a.a_d1 = r.a_d1; a.x_k0 = r.x_k0; a.x_n0 = r.x_n0;
  a.out = static_cast<double*>(r.out); a.ldo = r.ldo;
  a.xin = static_cast<const double*>(r.xin); a.ldx = r.ldx;
  a.alpha = r.alpha; a.beta = r.beta; a.c = r.c;
  a.use_beta = 0; a.band_lo = r.band_lo; a.band_hi = r.band_hi; a.band_shift = r.band_shift;
  a.band_map = r.band_map;
  a.a3d = r.a3d;
  const int grid = std::min(T, h->sm_budget > 0 ? std::min(h->sm_budget, h->num_sms) : h->num_sms);
  constexpr int S = dg_smem_bytes(DG_BN), SN = dg_smem_bytes(DG_BN_NARROW);
  if (narrow) {
    if (trans) dgemm_fused_kernel<true, DG_BN_NARROW><<<grid, DG_THREADS, SN, h->stream>>>(tA, tX, a, f);
    else dgemm_fused_kernel<false, DG_BN_NARROW><<<grid, DG_THREADS, SN, h->stream>>>(tA, tX, a, f);
  } else {
    if (trans) dgemm_fused_kernel<true><<<grid, DG_THREADS, S, h->stream>>>(tA, tX, a, f);
    else dgemm_fused_kernel<false><<<grid, DG_THREADS, S, h->stream>>>(tA, tX, a, f);
  }
  CUDA_TRY(cudaGetLastError());
  return CHASE_OK;
}

// Wave-quantisation tail plan for T equal-cost tiles of KT k-tiles on G co-resident CTAs: the
// last T_tail tiles as S split-K copies, (T_tail, S) minimising the modelled waves (T_tail = the
// partial last wave, or it plus one full wave); S = 1: no split (nothing gained).  T_tail <= cap.
static void plan_tail(int T, int KT, int G, int cap, int* S_out, int* tail_out) {
  *S_out = 1;
  *tail_out = 0;
  const int full = T / G, rem = T % G;
  if (rem == 0) return;
  double best_gain = 0.02;                 // in waves; below this the split is not worth it
  for (int extra = 0; extra <= std::min(1, full); ++extra) {
    const int tail = rem + extra * G;
    if (tail > cap) break;
    for (int S = 2; S <= 8; ++S) {
      if (KT < 2 * S || S * tail > TAIL_TILES_MAX) break;
      const int ktc = (KT + S - 1) / S;
      if ((KT + ktc - 1) / ktc != S) continue;   // S copies must all be non-empty
      const double waves = (double)((S * tail + G - 1) / G) / S;
      const double gain = (extra + 1) - waves;
      if (gain > best_gain) {
        best_gain = gain;
        *S_out = S;
        *tail_out = tail;
      }
    }
  }
}

// A big GEMM with its wave-quantisation tail split over K (gemm_tail.cuh): the plain kernel on
// the first T_main tiles of the raster, the last T_tail tiles as S split-K copies into tile-local
// partials, then the fixed-order sum + epilogue.  (T_tail, S) minimise the modelled waves
// (equal-cost tiles, one CTA per SM); no split when nothing is gained.
static chase_status_t run_gemm_tail(chase_handle_s* h, const GemmReq& g) {
  static const bool off = getenv("CHASE_NO_TAIL_SPLIT") != nullptr;   // A/B switches
  static const bool no_narrow = getenv("CHASE_NO_NARROW") != nullptr;
  const bool cplx = h->dt == CHASE_C128;
  if (g.tX_narrow && !no_narrow && !g.narrow && g.M > 0 && g.N > 0 && !g.col_shift && !g.diag_k &&
      !g.upper_only && g.k_split <= 1) {
    // ragged width: the N mod BN remainder columns as a narrow-tile GEMM when that pads less
    const int BNw = cplx ? ZG_BN : DG_BN, BNn = cplx ? ZG_BN_NARROW : DG_BN_NARROW;
    const int r = g.N % BNw;
    if (r != 0 && (r + BNn - 1) / BNn * BNn < BNw) {
      const size_t es = esize_of(h->dt);
      const int Nmain = g.N - r;
      if (Nmain > 0) {
        GemmReq m = g;
        m.N = Nmain;
        m.tX_narrow = nullptr;
        STATUS_TRY(run_gemm_tail(h, m));
      }
      GemmReq t = g;
      t.tX_narrow = nullptr;
      t.narrow = 1;
      t.tX = g.tX_narrow;
      t.N = r;
      t.x_n0 = g.x_n0 + Nmain;
      t.out = static_cast<char*>(g.out) + (size_t)Nmain * g.ldo * es;
      if (g.xin) t.xin = static_cast<const char*>(g.xin) + (size_t)Nmain * g.ldx * es;
      if (Nmain > 0) h->launches[g.conj ? CAT_HEMM_ODD : CAT_HEMM_EVEN] += 1;
      return run_gemm_tail(h, t);
    }
  }
  if (off || g.M <= 0 || g.N <= 0 || g.col_shift || g.diag_k || g.upper_only || g.abort_flag ||
      g.k_split > 1 || !h->tailws)
    return run_gemm(h, g);
  const int BM = cplx ? ZG_BM : DG_BM, BK = cplx ? ZG_BK : DG_BKT;
  const int BN = cplx ? (g.narrow ? ZG_BN_NARROW : ZG_BN) : (g.narrow ? DG_BN_NARROW : DG_BN);
  const int T = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN);
  const int SMS = h->num_sms, KT = (g.K + BK - 1) / BK;
  int bS, btail;
  plan_tail(T, KT, SMS, TAIL_TILES_MAX, &bS, &btail);
  if (bS == 1) return run_gemm(h, g);
  const int tmain = T - btail;
  if (tmain > 0) {
    GemmReq m = g;
    m.grid_tiles = tmain;
    STATUS_TRY(run_gemm(h, m));
  }
  GemmReq t = g;
  t.k_split = bS;
  t.tail_tiles = btail;
  t.tile_offset = tmain;
  t.out = h->tailws;
  t.ldo = BM;
  t.alpha = 1.0; t.beta = 0.0; t.c = 0.0; t.use_beta = 0;
  t.band_lo = t.band_hi = 0; t.band_shift = 0; t.band_map = nullptr;
  STATUS_TRY(run_gemm(h, t));
  TailArgs ta{bS, btail, tmain, g.M, g.N, (long long)g.ldo, (long long)g.ldx, g.alpha, g.beta, g.c,
              g.use_beta, g.band_lo, g.band_hi, g.band_shift, g.band_map};
  if (cplx && !g.narrow)
    gemm_tail_epilogue_kernel<double2, ZG_BM, ZG_BN, ZG_GROUP_M><<<btail, 256, 0, h->stream>>>(
        reinterpret_cast<const double2*>(h->tailws), static_cast<double2*>(g.out),
        static_cast<const double2*>(g.xin), ta);
  else if (cplx)
    gemm_tail_epilogue_kernel<double2, ZG_BM, ZG_BN_NARROW, ZG_GROUP_M><<<btail, 256, 0, h->stream>>>(
        reinterpret_cast<const double2*>(h->tailws), static_cast<double2*>(g.out),
        static_cast<const double2*>(g.xin), ta);
  else if (!g.narrow)
    gemm_tail_epilogue_kernel<double, DG_BM, DG_BN, DG_GROUP_M><<<btail, 256, 0, h->stream>>>(
        reinterpret_cast<const double*>(h->tailws), static_cast<double*>(g.out),
        static_cast<const double*>(g.xin), ta);
  else
    gemm_tail_epilogue_kernel<double, DG_BM, DG_BN_NARROW, DG_GROUP_M><<<btail, 256, 0, h->stream>>>(
        reinterpret_cast<const double*>(h->tailws), static_cast<double*>(g.out),
        static_cast<const double*>(g.xin), ta);
  CUDA_TRY(cudaGetLastError());
  h->launches[g.conj ? CAT_HEMM_ODD : CAT_HEMM_EVEN] += 2;
  return CHASE_OK;
}

static chase_status_t launch_zgemm_fused(chase_handle_s* h, bool conj, const CUtensorMap& tA,
                                         const CUtensorMap& tX, const GemmReq& r,
                                         const FusedArgs& f, int T, bool narrow) {
  if (r.M <= 0 || r.N <= 0) return CHASE_OK;
  if (h->dt == CHASE_R64) return launch_dgemm_fused(h, conj, tA, tX, r, f, T, narrow);
  ZGemmArgs a{};
  a.M = r.M; a.N = r.N; a.K = r.K;
  a.a_d0 = r.a_d0; a.a_d1 = r.a_d1; a.x_k0 = r.x_k0; a.x_n0 = r.x_n0;
  a.out = static_cast<double2*>(r.out); a.ldo = r.ldo;
  a.xin = static_cast<const double2*>(r.xin); a.ldx = r.ldx;
  a.alpha = r.alpha; a.beta = r.beta; a.c = r.c;
  a.use_beta = 0; a.band_lo = r.band_lo; a.band_hi = r.band_hi; a.band_shift = r.band_shift;
  a.band_map = r.band_map;
  a.a3d = r.a3d;
  const int grid = std::min(T, h->sm_budget > 0 ? std::min(h->sm_budget, h->num_sms) : h->num_sms);
  constexpr int S = ZG_SMEM_BYTES, SN = zg_smem_bytes(ZG_BN_NARROW);
  if (narrow) {
    if (conj) zgemm_fused_kernel<true, ZG_BN_NARROW><<<grid, ZG_THREADS, SN, h->stream>>>(tA, tX, a, f);
    else zgemm_fused_kernel<false, ZG_BN_NARROW><<<grid, ZG_THREADS, SN, h->stream>>>(tA, tX, a, f);
  } else {
    if (conj) zgemm_fused_kernel<true><<<grid, ZG_THREADS, S, h->stream>>>(tA, tX, a, f);
    else zgemm_fused_kernel<false><<<grid, ZG_THREADS, S, h->stream>>>(tA, tX, a, f);
  }
  CUDA_TRY(cudaGetLastError());
  return CHASE_OK;
}

// Tensor maps for the three roles a matrix plays in the GEMM (box shapes of zgemm / dgemm).
enum MapRole { ROLE_A_NOTRANS, ROLE_A_TRANS, ROLE_X, ROLE_X_NARROW };
// 3D view of a column-major matrix for the NoTrans A tile: dims {one 128-byte row piece,
// columns, row pieces} so one TMA box fills the whole BM x BK tile.  Only valid when every
// column has room for whole 128-byte pieces (ld >= rows rounded up to a piece), since TMA
// bounds-checks per dimension and the last piece may run past the column's rows.
static chase_status_t make_map_3d(CUtensorMap* m, const void* base, int64_t rows, int64_t cols,
                                  int64_t ld, int esize, int box_k, int box_pieces) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return CHASE_ECUDA;
  const int piece = 128 / esize;                       // elements per 128-byte row piece
  cuuint64_t dims[3] = {16, (cuuint64_t)cols, (cuuint64_t)((rows + piece - 1) / piece)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * esize), 128};
  cuuint32_t box[3] = {16, (cuuint32_t)box_k, (cuuint32_t)box_pieces};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? CHASE_OK : CHASE_ECUDA;
}

static chase_status_t make_role_map(const chase_handle_s* h, CUtensorMap* m, const void* base,
                                    int64_t rows, int64_t cols, int64_t ld, MapRole role,
                                    int* a3d = nullptr) {
  const int es = (int)esize_of(h->dt);
  if (a3d) *a3d = 0;
  if (role == ROLE_A_NOTRANS && a3d && !g_disable_a3d) {
    const int piece = 128 / es;
    const int64_t rows_up = (rows + piece - 1) / piece * piece;
    if (ld >= rows_up &&
        make_map_3d(m, base, rows, cols, ld, es, es == 16 ? 8 : DG_BK,
                    es == 16 ? ZG_BM / 8 : DG_BM / 16) == CHASE_OK) {
      *a3d = 1;
      return CHASE_OK;
    }
  }
  if (h->dt == CHASE_C128) {
    const int bc = role == ROLE_A_NOTRANS ? 8 : role == ROLE_A_TRANS ? ZG_BM
                   : role == ROLE_X_NARROW ? ZG_BN_NARROW : ZG_BN;
    return make_map(m, base, rows, cols, ld, 16, 8, bc);
  }
  const int bc = role == ROLE_A_NOTRANS ? DG_BK : role == ROLE_A_TRANS ? DG_BM
                 : role == ROLE_X_NARROW ? DG_BN_NARROW : DG_BN;
  return make_map(m, base, rows, cols, ld, 8, 16, bc);
}

static chase_status_t allreduce(chase_handle_s* h, void* buf, size_t elems, ncclComm_t comm) {
  ProfScope ps(h, CAT_ALLREDUCE, 0);
  const size_t nd = elems * (h->dt == CHASE_C128 ? 2 : 1);
  NCCL_TRY(ncclAllReduce(buf, buf, nd, ncclDouble, ncclSum, comm, h->stream));
  return CHASE_OK;
}

// Column-by-column AllReduce of a strided block (rows n_r of each column), one NCCL group.
static chase_status_t allreduce_cols(chase_handle_s* h, void* buf, int64_t rows, int64_t ld,
                                     int64_t cols, ncclComm_t comm) {
  ProfScope ps(h, CAT_ALLREDUCE, 0);
  const size_t es = esize_of(h->dt), per = es / 8;
  NCCL_TRY(ncclGroupStart());
  for (int64_t j = 0; j < cols; ++j) {
    char* p = static_cast<char*>(buf) + (size_t)j * ld * es;
    NCCL_TRY(ncclAllReduce(p, p, (size_t)rows * per, ncclDouble, ncclSum, comm, h->stream));
  }
  NCCL_TRY(ncclGroupEnd());
  return CHASE_OK;
}

// ==================================================================== SPMD argument check
// Collective calls need identical scalar arguments on every rank (include/chase.h).  With
// CHASE_SPMD_CHECK=1 in the environment (or a -DCHASE_DEBUG build) the call hashes them (FNV-1a
// over the raw bytes) and compares min and max of the hash over the world communicator; a
// mismatch returns CHASE_EINVAL on every rank before any device work.  Costs two tiny
// AllReduces and a stream synchronisation, so it is off by default.
static bool spmd_check_enabled() {
#ifdef CHASE_DEBUG
  return true;
#else
  static const bool on = getenv("CHASE_SPMD_CHECK") != nullptr && atoi(getenv("CHASE_SPMD_CHECK")) != 0;
  return on;
#endif
}
struct SpmdHash {
  uint64_t v = 1469598103934665603ull;
  void add(const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) v = (v ^ b[i]) * 1099511628211ull;
  }
  template <typename T> void add(const T& x) { add(&x, sizeof(T)); }
};
static chase_status_t spmd_verify(chase_handle_s* h, uint64_t hash) {
  if (!spmd_check_enabled() || h->world == nullptr) return CHASE_OK;
  uint64_t* d = reinterpret_cast<uint64_t*>(h->d_shift) + 1;   // scratch words after the shift
  uint64_t hv[2] = {hash, hash};
  CUDA_TRY(cudaMemcpyAsync(d, hv, 16, cudaMemcpyHostToDevice, h->stream));
  NCCL_TRY(ncclGroupStart());
  NCCL_TRY(ncclAllReduce(d, d, 1, ncclUint64, ncclMin, h->world, h->stream));
  NCCL_TRY(ncclAllReduce(d + 1, d + 1, 1, ncclUint64, ncclMax, h->world, h->stream));
  NCCL_TRY(ncclGroupEnd());
  CUDA_TRY(cudaMemcpyAsync(hv, d, 16, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (hv[0] != hv[1]) {
    fprintf(stderr, "[chase] SPMD check: arguments differ across ranks\n");
    return CHASE_EINVAL;
  }
  return CHASE_OK;
}

// ==================================================================== fused-comm workspace
// Symmetric region (identical size and layout on every rank, peer-mapped by the caller):
//   Cw  C-layout working block  pad(ceil(N/p)) x n_max      (filter even-step outputs)
//   Bw  B-layout working block  pad(ceil(N/q)) x n_max      (filter odd-step outputs)
//   P   partial tiles           pad(max rows)  x n_max
//   flags [tile * m + src] u32  (tiles of the largest step) x max(p, q), one array per parity
//   done  u64 delivery counter, err i32, tile-scheduler counter
//   tailp FUSED_TAIL_SLOTS slots x max(p, q) sub-slots of split-K tail partial tiles,
//         tflags [slot][src] (fused_tail.cuh)
struct FusedLayout {
  int64_t ldc, ldb, ldpo, ldpe;
  size_t cw, bw, po, pe, flags, done, err, ctr, tailp, tflags, total;
  int64_t tiles_max;
};
// Staging areas by step parity (odd steps: p slots of B-layout rows, even: q slots of C-layout
// rows) so a member pushing step s+1 partials never overwrites slots still being summed for s.
static FusedLayout fused_layout(const chase_handle_s* h) {
  FusedLayout L;
  int64_t nr_max = (h->N + h->p - 1) / h->p, nc_max = (h->N + h->q - 1) / h->q;
  if (h->nb > 0) {                       // block-cyclic: largest local block over the grid
    std::vector<int64_t> v;
    nr_max = nc_max = 0;
    for (int k = 0; k < h->p; ++k) {
      cyclic_indices(h->N, h->p, k, h->nb, &v);
      nr_max = std::max<int64_t>(nr_max, (int64_t)v.size());
    }
    for (int k = 0; k < h->q; ++k) {
      cyclic_indices(h->N, h->q, k, h->nb, &v);
      nc_max = std::max<int64_t>(nc_max, (int64_t)v.size());
    }
  }
  const int64_t rows_max = std::max(nr_max, nc_max);
  L.ldc = pad_ld(nr_max);
  L.ldb = pad_ld(nc_max);
  L.ldpo = L.ldb;
  L.ldpe = L.ldc;
  // tiles of the largest step (complex 128 x 64 tiles; real ones are no smaller) plus the narrow
  // remainder tiles of a split step (at most 4 per m-tile)
  L.tiles_max = ((rows_max + ZG_BM - 1) / ZG_BM) * ((h->n_max + ZG_BN - 1) / ZG_BN + 4);
  size_t off = 0;
  L.cw = off;
  off += align256((size_t)L.ldc * h->n_max * 16);
  L.bw = off;
  off += align256((size_t)L.ldb * h->n_max * 16);
  L.po = off;
  off += align256((size_t)h->p * L.ldpo * h->n_max * 16);
  L.pe = off;
  off += align256((size_t)h->q * L.ldpe * h->n_max * 16);
  L.flags = off;
  off += align256((size_t)2 * L.tiles_max * std::max(h->p, h->q) * sizeof(unsigned));
  L.done = off;
  off += 256;
  L.err = off;
  off += 256;
  L.ctr = off;                                          // dynamic tile-scheduler counter
  off += 256;
  L.tailp = off;                                        // split-K tail partials (fused_tail.cuh)
  off += align256((size_t)FUSED_TAIL_SLOTS * std::max(h->p, h->q) * FUSED_TAIL_TILES * 128 * 128 * 8);
  L.tflags = off;                                       // tail flags [slot][src]
  off += align256((size_t)FUSED_TAIL_SLOTS * FUSED_MAX_MEMBERS * sizeof(unsigned));
  L.total = off;
  return L;
}

// ==================================================================== kernel preloading
// Load (and size the dynamic shared memory of) every kernel of the filter and CholeskyQR paths
// once per process, before the first launch.  Under CUDA lazy module loading the first launch
// of a kernel loads its module and may wait for the device to go idle; a fused kernel spinning
// on a peer that is itself blocked in such a load (several ranks of a virtual grid in one
// process) would wait for nothing until its timeout, and a first-use load inside a timed
// region would be charged to it.
static chase_status_t preload_kernels() {
  static std::once_flag once;
  static chase_status_t status = CHASE_OK;
  std::call_once(once, [] {
    auto smem = [](const void* k, int bytes) {
      cudaFuncAttributes a;
      if (cudaFuncGetAttributes(&a, k) != cudaSuccess) return false;
      return bytes == 0 || cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess;
    };
    bool ok = true;
    ok &= smem((const void*)zgemm_kernel<true>, ZG_SMEM_BYTES);
    ok &= smem((const void*)zgemm_kernel<false>, ZG_SMEM_BYTES);
    ok &= smem((const void*)zgemm_kernel<true, true>, ZG_SMEM_BYTES);
    ok &= smem((const void*)zgemm_kernel<false, true>, ZG_SMEM_BYTES);
    ok &= smem((const void*)dgemm_kernel<true>, dg_smem_bytes(DG_BN));
    ok &= smem((const void*)dgemm_kernel<false>, dg_smem_bytes(DG_BN));
    ok &= smem((const void*)dgemm_kernel<true, true>, dg_smem_bytes(DG_BN));
    ok &= smem((const void*)dgemm_kernel<false, true>, dg_smem_bytes(DG_BN));
    ok &= smem((const void*)zgemm_fused_kernel<true>, ZG_SMEM_BYTES);
    ok &= smem((const void*)zgemm_fused_kernel<false>, ZG_SMEM_BYTES);
    ok &= smem((const void*)dgemm_fused_kernel<true>, dg_smem_bytes(DG_BN));
    ok &= smem((const void*)dgemm_fused_kernel<false>, dg_smem_bytes(DG_BN));
    ok &= smem((const void*)dgemm_fused_kernel<true, DG_BN_NARROW>, dg_smem_bytes(DG_BN_NARROW));
    ok &= smem((const void*)dgemm_fused_kernel<false, DG_BN_NARROW>, dg_smem_bytes(DG_BN_NARROW));
    ok &= smem((const void*)zgemm_fused_kernel<true, ZG_BN_NARROW>, zg_smem_bytes(ZG_BN_NARROW));
    ok &= smem((const void*)zgemm_fused_kernel<false, ZG_BN_NARROW>, zg_smem_bytes(ZG_BN_NARROW));
    ok &= smem((const void*)fused_wait_kernel, 0);
    ok &= smem((const void*)zgemm_kernel<true, false, ZG_BN_NARROW>, zg_smem_bytes(ZG_BN_NARROW));
    ok &= smem((const void*)zgemm_kernel<false, false, ZG_BN_NARROW>, zg_smem_bytes(ZG_BN_NARROW));
    ok &= smem((const void*)zgemm_kernel<true, true, ZG_BN_NARROW>, zg_smem_bytes(ZG_BN_NARROW));
    ok &= smem((const void*)zgemm_kernel<false, true, ZG_BN_NARROW>, zg_smem_bytes(ZG_BN_NARROW));
    ok &= smem((const void*)dgemm_kernel<true, false, DG_BN_NARROW>, dg_smem_bytes(DG_BN_NARROW));
    ok &= smem((const void*)dgemm_kernel<false, false, DG_BN_NARROW>, dg_smem_bytes(DG_BN_NARROW));
    ok &= smem((const void*)dgemm_kernel<true, true, DG_BN_NARROW>, dg_smem_bytes(DG_BN_NARROW));
    ok &= smem((const void*)dgemm_kernel<false, true, DG_BN_NARROW>, dg_smem_bytes(DG_BN_NARROW));
    ok &= smem((const void*)zgemm_kernel<false, false, ZG_BN, true>, ZG_SMEM_BYTES);
    ok &= smem((const void*)dgemm_kernel<false, false, DG_BN, true>, dg_smem_bytes(DG_BN));
    ok &= smem((const void*)gemm_tail_epilogue_kernel<double2, ZG_BM, ZG_BN_NARROW, ZG_GROUP_M>, 0);
    ok &= smem((const void*)gemm_tail_epilogue_kernel<double, DG_BM, DG_BN_NARROW, DG_GROUP_M>, 0);
    ok &= smem((const void*)gemm_tail_epilogue_kernel<double2, ZG_BM, ZG_BN, ZG_GROUP_M>, 0);
    ok &= smem((const void*)gemm_tail_epilogue_kernel<double, DG_BM, DG_BN, DG_GROUP_M>, 0);
    ok &= smem((const void*)fused_tail_sync_kernel, 0);
    ok &= smem((const void*)fused_tail_publish_kernel<double2, ZG_BM, ZG_BN, ZG_GROUP_M>, 0);
    ok &= smem((const void*)fused_tail_publish_kernel<double2, ZG_BM, ZG_BN_NARROW, ZG_GROUP_M>, 0);
    ok &= smem((const void*)fused_tail_publish_kernel<double, DG_BM, DG_BN, DG_GROUP_M>, 0);
    ok &= smem((const void*)fused_tail_publish_kernel<double, DG_BM, DG_BN_NARROW, DG_GROUP_M>, 0);
    ok &= smem((const void*)fused_tail_reduce_kernel<double2, ZG_BM, ZG_BN, ZG_GROUP_M>, 0);
    ok &= smem((const void*)fused_tail_reduce_kernel<double2, ZG_BM, ZG_BN_NARROW, ZG_GROUP_M>, 0);
    ok &= smem((const void*)fused_tail_reduce_kernel<double, DG_BM, DG_BN, DG_GROUP_M>, 0);
    ok &= smem((const void*)fused_tail_reduce_kernel<double, DG_BM, DG_BN_NARROW, DG_GROUP_M>, 0);
    if (!ok) {
      fprintf(stderr, "[chase] kernel preload failed: %s\n", cudaGetErrorString(cudaGetLastError()));
      status = CHASE_ECUDA;
    }
  });
  return status;
}

// ==================================================================== schedule (pure)
static chase_status_t validate_degrees(int64_t ncols, const int32_t* degrees) {
  if (!degrees) return CHASE_EINVAL;
  for (int64_t j = 0; j < ncols; ++j) {
    const int32_t d = degrees[j];
    if (d < 2 || (d % 2) != 0) return CHASE_EDEGREE;
    if (j > 0 && d < degrees[j - 1]) return CHASE_EDEGREE;
  }
  return CHASE_OK;
}

// The per-step schedule of rank (myrow, mycol): active width, offset, communicator, message
// size, and the rank's share of the -cI shift (band) and of the beta term (use_beta).
struct Geom {
  int64_t n_r, n_c, r0, c0;
  int myrow, mycol;
  int64_t nb = 0;   // block-cyclic: the band is irregular (device maps); recorded as [-1, -1)
};
static void build_schedule(const Geom& gm, int64_t ncols, const int32_t* degrees,
                           std::vector<chase_step_record_t>* rec, int64_t* matvecs) {
  const int32_t D = degrees[ncols - 1];
  rec->assign(D, chase_step_record_t{});
  int64_t mv = 0;
  for (int64_t j = 0; j < ncols; ++j) mv += degrees[j];
  int64_t first = 0;  // first column with d_j >= s (degrees sorted)
  for (int32_t s = 1; s <= D; ++s) {
    while (first < ncols && degrees[first] < s) ++first;
    chase_step_record_t& r = (*rec)[s - 1];
    const bool odd = (s % 2 == 1);
    r.k = (int32_t)(ncols - first);
    r.off = (int32_t)first;
    r.comm = odd ? 0 : 1;
    r.elems = (int64_t)r.k * (odd ? gm.n_c : gm.n_r);
    if (gm.nb > 0) {
      r.band_lo = r.band_hi = -1;
      r.use_beta = odd ? ((gm.myrow == 0 && s > 1) ? 1 : 0) : (gm.mycol == 0 ? 1 : 0);
    } else if (odd) {   // output rows = B_j rows (global c0 + row); diagonal rows also in [r0, r0+n_r)
      r.band_lo = (int32_t)std::max<int64_t>(0, gm.r0 - gm.c0);
      r.band_hi = (int32_t)std::max<int64_t>(r.band_lo, std::min<int64_t>(gm.n_c, gm.r0 + gm.n_r - gm.c0));
      r.use_beta = (gm.myrow == 0 && s > 1) ? 1 : 0;
    } else {     // output rows = C_i rows (global r0 + row); diagonal rows also in [c0, c0+n_c)
      r.band_lo = (int32_t)std::max<int64_t>(0, gm.c0 - gm.r0);
      r.band_hi = (int32_t)std::max<int64_t>(r.band_lo, std::min<int64_t>(gm.n_r, gm.c0 + gm.n_c - gm.r0));
      r.use_beta = (gm.mycol == 0) ? 1 : 0;
    }
  }
  *matvecs = mv;
}

// ==================================================================== C-ABI
extern "C" {

const char* chase_status_string(chase_status_t s) {
  switch (s) {
    case CHASE_OK: return "CHASE_OK";
    case CHASE_EINVAL: return "CHASE_EINVAL: invalid argument";
    case CHASE_EDEGREE: return "CHASE_EDEGREE: degrees must be even, >= 2 and non-decreasing";
    case CHASE_EBOUNDS: return "CHASE_EBOUNDS: e <= 0 or mu_1 inside the damped interval";
    case CHASE_ECHOL: return "CHASE_ECHOL: Cholesky factorisation failed";
    case CHASE_ECUDA: return "CHASE_ECUDA: CUDA failure";
    case CHASE_ENCCL: return "CHASE_ENCCL: NCCL failure";
    case CHASE_ENOMEM: return "CHASE_ENOMEM: workspace missing or too small";
    case CHASE_ESTATE: return "CHASE_ESTATE: invalid call sequence";
    case CHASE_ENOCONV: return "CHASE_ENOCONV: not converged within max_iter (partial results)";
  }
  return "CHASE_?: unknown status";
}

chase_status_t chase_get_unique_id(uint8_t id[128]) {
  if (!id) return CHASE_EINVAL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId uid;
  NCCL_TRY(ncclGetUniqueId(&uid));
  memcpy(id, &uid, 128);
  return CHASE_OK;
}

chase_status_t chase_block_dims(int64_t N, int p, int q, int i, int j, int64_t* n_r,
                                int64_t* n_c, int64_t* r0, int64_t* c0) {
  if (N < 1 || p < 1 || q < 1 || i < 0 || i >= p || j < 0 || j >= q || !n_r || !n_c || !r0 ||
      !c0 || p > N || q > N)
    return CHASE_EINVAL;
  block_part(N, p, i, n_r, r0);
  block_part(N, q, j, n_c, c0);
  return CHASE_OK;
}

chase_status_t chase_create(chase_handle_t* out, chase_dtype_t dt, int64_t N, int64_t n_max,
                            int p, int q, int myrow, int mycol, const uint8_t id[128], int device,
                            void* cuda_stream) {
  return chase_create_cyclic(out, dt, N, n_max, p, q, myrow, mycol, 0, id, device, cuda_stream);
}

}  // extern "C"

static chase_status_t create_handle(chase_handle_t* out, chase_dtype_t dt, int64_t N, int64_t n_max,
                                    int p, int q, int myrow, int mycol, int64_t nb,
                                    const uint8_t id[128], int device, void* cuda_stream, bool virt) {
  if (!out) return CHASE_EINVAL;
  if (nb < 0) return CHASE_EINVAL;
  *out = nullptr;
  if (dt != CHASE_R64 && dt != CHASE_C128) return CHASE_EINVAL;
  if (N < 1 || n_max < 1 || n_max > N || N > (int64_t)INT32_MAX) return CHASE_EINVAL;
  if (p < 1 || q < 1 || myrow < 0 || myrow >= p || mycol < 0 || mycol >= q) return CHASE_EINVAL;
  if (p > N || q > N) return CHASE_EINVAL;
  if (p * q > 1 && !id && !virt) return CHASE_EINVAL;
  chase_handle_s* h = new chase_handle_s();
  h->virt = virt;
  h->dt = dt;
  h->N = N;
  h->n_max = n_max;
  h->p = p;
  h->q = q;
  h->myrow = myrow;
  h->mycol = mycol;
  h->nb = nb;
  if (nb == 0) {
    block_part(N, p, myrow, &h->n_r, &h->r0);
    block_part(N, q, mycol, &h->n_c, &h->c0);
    h->voff = h->r0;
    for (int64_t l = 0; l < h->n_r; ++l) h->rows_g.push_back(h->r0 + l);
    for (int64_t l = 0; l < h->n_c; ++l) h->cols_g.push_back(h->c0 + l);
  } else {
    cyclic_indices(N, p, myrow, nb, &h->rows_g);
    cyclic_indices(N, q, mycol, nb, &h->cols_g);
    h->n_r = (int64_t)h->rows_g.size();
    h->n_c = (int64_t)h->cols_g.size();
    h->r0 = h->c0 = -1;
    if (h->n_r == 0 || h->n_c == 0) {
      delete h;
      return CHASE_EINVAL;                    // every grid row/column must own at least one block
    }
    std::vector<int64_t> other;
    for (int i2 = 0; i2 < myrow; ++i2) {
      cyclic_indices(N, p, i2, nb, &other);
      h->voff += (int64_t)other.size();
    }
  }
  h->device = device;
  h->stream = static_cast<cudaStream_t>(cuda_stream);
  if (cudaSetDevice(device) != cudaSuccess || cudaMallocHost(&h->h_info, sizeof(int)) != cudaSuccess ||
      cudaMallocHost(&h->h_shift, sizeof(double)) != cudaSuccess) {
    delete h;
    return CHASE_ECUDA;
  }
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (preload_kernels() != CHASE_OK) {
    chase_destroy(h);
    return CHASE_ECUDA;
  }
  if (p * q > 1 && !virt) {
    ncclUniqueId uid;
    memcpy(&uid, id, 128);
    const int rank = myrow * q + mycol;
    ncclResult_t r = ncclCommInitRank(&h->world, p * q, uid, rank);
    if (r == ncclSuccess) r = ncclCommSplit(h->world, myrow, mycol, &h->rcomm, nullptr);
    if (r == ncclSuccess) r = ncclCommSplit(h->world, mycol, myrow, &h->ccomm, nullptr);
    if (r != ncclSuccess) {
      fprintf(stderr, "[chase] NCCL setup failed: %s\n", ncclGetErrorString(r));
      chase_destroy(h);
      return CHASE_ENCCL;
    }
  }
  *out = h;
  return CHASE_OK;
}

extern "C" {

chase_status_t chase_create_cyclic(chase_handle_t* out, chase_dtype_t dt, int64_t N, int64_t n_max,
                                   int p, int q, int myrow, int mycol, int64_t nb,
                                   const uint8_t id[128], int device, void* cuda_stream) {
  return create_handle(out, dt, N, n_max, p, q, myrow, mycol, nb, id, device, cuda_stream, false);
}

chase_status_t chase_create_virtual(chase_handle_t* out, chase_dtype_t dt, int64_t N, int64_t n_max,
                                    int p, int q, int myrow, int mycol, int64_t nb, int device,
                                    void* cuda_stream) {
  return create_handle(out, dt, N, n_max, p, q, myrow, mycol, nb, nullptr, device, cuda_stream, true);
}

chase_status_t chase_set_fused_mode(chase_handle_t h, int32_t mode, int32_t sm_budget) {
  if (!h || (mode != 0 && mode != 1) || sm_budget < 0) return CHASE_EINVAL;
  h->fused_mode = mode;
  h->sm_budget = sm_budget;
  return CHASE_OK;
}

chase_status_t chase_set_stream(chase_handle_t h, void* cuda_stream) {
  if (!h) return CHASE_EINVAL;
  h->stream = static_cast<cudaStream_t>(cuda_stream);
  return CHASE_OK;
}

chase_status_t chase_local_dims(chase_handle_t h, int64_t* n_r, int64_t* n_c, int64_t* r0,
                                int64_t* c0) {
  if (!h || !n_r || !n_c || !r0 || !c0) return CHASE_EINVAL;
  *n_r = h->n_r;
  *n_c = h->n_c;
  *r0 = h->r0;
  *c0 = h->c0;
  return CHASE_OK;
}

chase_status_t chase_local_indices(chase_handle_t h, int64_t* rows, int64_t* cols) {
  if (!h) return CHASE_EINVAL;
  if (rows) memcpy(rows, h->rows_g.data(), h->rows_g.size() * sizeof(int64_t));
  if (cols) memcpy(cols, h->cols_g.data(), h->cols_g.size() * sizeof(int64_t));
  return CHASE_OK;
}

chase_status_t chase_cyclic_indices(int64_t N, int P, int k, int64_t nb, int64_t* idx,
                                    int64_t* count) {
  if (N < 1 || P < 1 || k < 0 || k >= P || nb < 1 || !count) return CHASE_EINVAL;
  std::vector<int64_t> v;
  cyclic_indices(N, P, k, nb, &v);
  *count = (int64_t)v.size();
  if (idx) memcpy(idx, v.data(), v.size() * sizeof(int64_t));
  return CHASE_OK;
}

chase_status_t chase_workspace_size(chase_handle_t h, size_t* bytes) {
  if (!h || !bytes) return CHASE_EINVAL;
  *bytes = ws_layout(h).total;
  return CHASE_OK;
}

chase_status_t chase_set_workspace(chase_handle_t h, void* dptr, size_t bytes) {
  if (!h || !dptr || (reinterpret_cast<uintptr_t>(dptr) & 255) != 0) return CHASE_EINVAL;
  const WsLayout L = ws_layout(h);
  if (bytes < L.total) return CHASE_ENOMEM;
  char* base = static_cast<char*>(dptr);
  h->ws = dptr;
  h->ws_bytes = bytes;
  h->Bws = base + L.b;
  h->Gws = base + L.g;
  h->Wws = base + L.w;
  h->Rinv = base + L.rinv;
  h->Rfws = base + L.rf;
  h->B2ws = base + L.b2;
  h->eigws = base + L.eig;
  h->c2ws = base + L.c2;
  h->lanws = base + L.lan;
  h->hhws = base + L.hh;
  h->tailws = base + L.tail;
  h->d_ritz = reinterpret_cast<double*>(base + L.ritz);
  h->d_nrm = reinterpret_cast<double*>(base + L.nrm);
  if (h->nb > 0) {
    // block-cyclic maps: band of -cI for both layouts and the residual B2 gather/scatter lists
    int* maps = reinterpret_cast<int*>(base + L.maps);
    h->d_band_even = maps;
    h->d_band_odd = maps + h->n_r;
    h->d_b2_src = maps + h->n_r + h->n_c;
    h->d_b2_dst = maps + h->n_r + 2 * h->n_c;
    std::vector<int> band_even(h->n_r, -1), band_odd(h->n_c, -1), src, dst;
    std::vector<int64_t> pos_c(h->N, -1), pos_r(h->N, -1);
    for (int64_t l = 0; l < h->n_c; ++l) pos_c[h->cols_g[l]] = l;
    for (int64_t l = 0; l < h->n_r; ++l) pos_r[h->rows_g[l]] = l;
    for (int64_t l = 0; l < h->n_r; ++l) band_even[l] = (int)pos_c[h->rows_g[l]];
    for (int64_t l = 0; l < h->n_c; ++l) band_odd[l] = (int)pos_r[h->cols_g[l]];
    h->b2_seg.assign(1, 0);
    std::vector<int64_t> owner_rows;
    for (int i2 = 0; i2 < h->p; ++i2) {
      cyclic_indices(h->N, h->p, i2, h->nb, &owner_rows);
      std::vector<int64_t> opos(h->N, -1);
      for (int64_t l = 0; l < (int64_t)owner_rows.size(); ++l) opos[owner_rows[l]] = l;
      for (int64_t l = 0; l < h->n_c; ++l) {
        const int64_t g = h->cols_g[l];
        if (opos[g] >= 0) {
          src.push_back((int)opos[g]);
          dst.push_back((int)l);
        }
      }
      h->b2_seg.push_back((int64_t)src.size());
    }
    CUDA_TRY(cudaMemcpy(h->d_band_even, band_even.data(), h->n_r * sizeof(int), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(h->d_band_odd, band_odd.data(), h->n_c * sizeof(int), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(h->d_b2_src, src.data(), src.size() * sizeof(int), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(h->d_b2_dst, dst.data(), dst.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  h->d_info = reinterpret_cast<int*>(base + L.info);
  h->d_shift = reinterpret_cast<double*>(base + L.s);
  return CHASE_OK;
}

chase_status_t chase_fused_workspace_size(chase_handle_t h, size_t* bytes) {
  if (!h || !bytes) return CHASE_EINVAL;
  *bytes = fused_layout(h).total;
  return CHASE_OK;
}

chase_status_t chase_set_fused_workspace(chase_handle_t h, void* local, const uint64_t* peer_bases,
                                         int world) {
  if (!h) return CHASE_EINVAL;
  if (!local) {
    h->fused = false;
    h->fused_broken = false;
    return CHASE_OK;
  }
  if (world != h->p * h->q || !peer_bases || world > 64) return CHASE_EINVAL;
  const int me = h->myrow * h->q + h->mycol;
  if (peer_bases[me] != reinterpret_cast<uint64_t>(local)) return CHASE_EINVAL;
  if (h->p > FUSED_MAX_MEMBERS || h->q > FUSED_MAX_MEMBERS) return CHASE_EINVAL;
  for (int r = 0; r < world; ++r) {
    if (!peer_bases[r] || (peer_bases[r] & 255)) return CHASE_EINVAL;
    h->fz_base[r] = reinterpret_cast<char*>(peer_bases[r]);
  }
  h->world_size = world;
  const FusedLayout L = fused_layout(h);
  // flags, counters, error word and tail flags start at zero; the caller barriers all ranks
  // before use
  CUDA_TRY(cudaMemsetAsync(static_cast<char*>(local) + L.flags, 0, L.tailp - L.flags, h->stream));
  CUDA_TRY(cudaMemsetAsync(static_cast<char*>(local) + L.tflags, 0, L.total - L.tflags, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  CUDA_TRY(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device));
  h->d_err = reinterpret_cast<int*>(static_cast<char*>(local) + L.err);
  h->fused_ep = 0;
  h->fused_delivered = 0;
  h->fused_tail_k[0] = h->fused_tail_k[1] = 0;
  h->fused_broken = false;
  h->fused = true;
  return CHASE_OK;
}

chase_status_t chase_filter_schedule(int64_t N, int p, int q, int myrow, int mycol, int64_t ncols,
                                     const int32_t* degrees, int32_t max_steps,
                                     chase_step_record_t* rec, int32_t* nsteps,
                                     int64_t* matvecs) {
  int64_t n_r, n_c, r0, c0;
  STATUS_TRY(chase_block_dims(N, p, q, myrow, mycol, &n_r, &n_c, &r0, &c0));
  if (ncols < 1 || ncols > N || !nsteps) return CHASE_EINVAL;
  STATUS_TRY(validate_degrees(ncols, degrees));
  std::vector<chase_step_record_t> r;
  int64_t mv;
  build_schedule(Geom{n_r, n_c, r0, c0, myrow, mycol}, ncols, degrees, &r, &mv);
  *nsteps = (int32_t)r.size();
  if (matvecs) *matvecs = mv;
  if (rec) {
    if (max_steps < (int32_t)r.size()) return CHASE_EINVAL;
    memcpy(rec, r.data(), r.size() * sizeof(chase_step_record_t));
  }
  return CHASE_OK;
}

chase_status_t chase_filter_record(chase_handle_t h, int32_t max_steps, chase_step_record_t* rec,
                                   int32_t* nsteps, int64_t* matvecs) {
  if (!h || !nsteps) return CHASE_EINVAL;
  *nsteps = (int32_t)h->record.size();
  if (matvecs) *matvecs = h->last_matvecs;
  if (rec) {
    if (max_steps < (int32_t)h->record.size()) return CHASE_EINVAL;
    memcpy(rec, h->record.data(), h->record.size() * sizeof(chase_step_record_t));
  }
  return CHASE_OK;
}

// Eq.(1) with the S:362 scalars; odd steps H^H-side into B, even steps into C.
chase_status_t chase_filter(chase_handle_t h, const void* A_local, int64_t lda, void* V,
                            int64_t ldv, int64_t ncols, const int32_t* degrees, double c,
                            double e, const chase_bounds_t* bounds, chase_stats_t* stats) {
  Nvtx nv_("chase_filter");
  if (!h || !A_local || !V || !bounds) return CHASE_EINVAL;
  if (ncols < 1 || ncols > h->n_max) return CHASE_EINVAL;
  if (lda < h->n_r || ldv < h->n_r) return CHASE_EINVAL;
  if (!std::isfinite(c) || !std::isfinite(e) || !std::isfinite(bounds->mu_1)) return CHASE_EINVAL;
  STATUS_TRY(validate_degrees(ncols, degrees));
  if (!(e > 0.0)) return CHASE_EBOUNDS;
  const double t1 = (bounds->mu_1 - c) / e;
  if (!(t1 <= -1.0)) return CHASE_EBOUNDS;
  if (!h->ws) return CHASE_ESTATE;
  const size_t es = esize_of(h->dt);
  if ((reinterpret_cast<uintptr_t>(A_local) & 15) || (reinterpret_cast<uintptr_t>(V) & 15))
    return CHASE_EINVAL;
  if (((size_t)lda * es) % 16 || ((size_t)ldv * es) % 16) return CHASE_EINVAL;   // TMA pitch

  if (spmd_check_enabled()) {
    SpmdHash hs;
    hs.add(ncols);
    hs.add(degrees, (size_t)ncols * sizeof(int32_t));
    hs.add(c);
    hs.add(e);
    hs.add(*bounds);
    STATUS_TRY(spmd_verify(h, hs.v));
  }
  std::vector<chase_step_record_t> rec;
  int64_t mv;
  build_schedule(Geom{h->n_r, h->n_c, h->r0, h->c0, h->myrow, h->mycol, h->nb}, ncols, degrees, &rec, &mv);
  const int D = (int)rec.size();

  // recurrence scalars: alpha_1 = sigma_1/e, beta_1 = 0; alpha_s = 2 sigma_s/e,
  // beta_s = -sigma_{s-1} sigma_s
  std::vector<double> alpha(D), beta(D);
  const double sigma_1 = e / (bounds->mu_1 - c);
  double sigma = sigma_1;
  alpha[0] = sigma_1 / e;
  beta[0] = 0.0;
  for (int s = 2; s <= D; ++s) {
    const double sigma_prev = sigma;
    sigma = 1.0 / (2.0 / sigma_1 - sigma_prev);
    alpha[s - 1] = 2.0 * sigma / e;
    beta[s - 1] = -sigma_prev * sigma;
  }

  const int64_t n_r = h->n_r, n_c = h->n_c;
  // working buffers: NCCL mode filters V in place and uses the B workspace; fused mode runs in
  // the symmetric region (peers write their reduced tiles straight into it)
  // fused_mode 1 (chase_set_fused_mode): the fused kernel runs even for single-member steps
  // (its protocol with itself; makes the fused kernels testable on one GPU)
  const bool fused_self = h->fused_mode == 1;
  const bool fused = h->fused && (h->p > 1 || h->q > 1 || fused_self);
  if (h->fused && h->fused_broken) return CHASE_ESTATE;     // re-run chase_set_fused_workspace
  if (h->virt && !fused && h->p * h->q > 1) return CHASE_ESTATE;   // no NCCL on a virtual grid
  FusedLayout FL{};
  char* Cbuf = static_cast<char*>(V);
  int64_t ldc = ldv;
  char* Bbuf = static_cast<char*>(h->Bws);
  int64_t ldb = pad_ld(n_c);
  const int me_world = h->myrow * h->q + h->mycol;
  if (fused) {
    FL = fused_layout(h);
    Cbuf = h->fz_base[me_world] + FL.cw;
    ldc = FL.ldc;
    Bbuf = h->fz_base[me_world] + FL.bw;
    ldb = FL.ldb;
    CUDA_TRY(cudaMemcpy2DAsync(Cbuf, ldc * es, V, ldv * es, n_r * es, ncols,
                               cudaMemcpyDeviceToDevice, h->stream));
  }
  CUtensorMap tA_nt, tA_t, tC, tB, tCn, tBn;
  int a3d = 0;
  STATUS_TRY(make_role_map(h, &tA_nt, A_local, n_r, n_c, lda, ROLE_A_NOTRANS, &a3d));
  STATUS_TRY(make_role_map(h, &tA_t, A_local, n_r, n_c, lda, ROLE_A_TRANS));
  STATUS_TRY(make_role_map(h, &tC, Cbuf, n_r, ncols, ldc, ROLE_X));
  STATUS_TRY(make_role_map(h, &tB, Bbuf, n_c, ncols, ldb, ROLE_X));
  STATUS_TRY(make_role_map(h, &tCn, Cbuf, n_r, ncols, ldc, ROLE_X_NARROW));   // remainder columns
  STATUS_TRY(make_role_map(h, &tBn, Bbuf, n_c, ncols, ldb, ROLE_X_NARROW));

  for (int s = 1; s <= D; ++s) {
    const chase_step_record_t& r = rec[s - 1];
    const bool odd = (s % 2 == 1);
    GemmReq g{};
    g.alpha = alpha[s - 1];
    g.beta = beta[s - 1];
    g.c = c;
    g.upper_only = 0;
    g.abort_flag = nullptr;
    g.a3d = 0;
    g.x_k0 = 0;
    g.x_n0 = r.off;
    g.a_d0 = 0;
    g.a_d1 = 0;
    g.N = r.k;
    if (odd) {
      // B_j = alpha (A_ij^H C_i - c band(C_i)) + [i == 0, s > 1] beta B_j
      g.conj = true;
      g.tA = &tA_t;
      g.tX = &tC;
      g.tX_narrow = &tCn;
      g.M = (int)n_c;
      g.K = (int)n_r;
      g.out = Bbuf + (size_t)r.off * ldb * es;
      g.ldo = ldb;
      g.xin = Cbuf + (size_t)r.off * ldc * es;
      g.ldx = ldc;
      g.band_lo = r.band_lo;
      g.band_hi = r.band_hi;
      g.band_shift = (int)(h->c0 - h->r0);   // input C row = output B row + c0 - r0
      g.band_map = h->nb > 0 ? h->d_band_odd : nullptr;
      g.use_beta = r.use_beta;
    } else {
      // C_i = alpha (A_ij B_j - c band(B_j)) + [j == 0] beta C_i
      g.conj = false;
      g.tA = &tA_nt;
      g.a3d = a3d;
      g.tX = &tB;
      g.tX_narrow = &tBn;
      g.M = (int)n_r;
      g.K = (int)n_c;
      g.out = Cbuf + (size_t)r.off * ldc * es;
      g.ldo = ldc;
      g.xin = Bbuf + (size_t)r.off * ldb * es;
      g.ldx = ldb;
      g.band_lo = r.band_lo;
      g.band_hi = r.band_hi;
      g.band_shift = (int)(h->r0 - h->c0);   // input B row = output C row + r0 - c0
      g.band_map = h->nb > 0 ? h->d_band_even : nullptr;
      g.use_beta = r.use_beta;
    }
    const int m = odd ? h->p : h->q;
    if (fused && (m > 1 || fused_self)) {
      // one kernel: HEMM + AllReduce over the step's communicator through peer memory
      FusedArgs f{};
      f.m = m;
      f.me = odd ? h->myrow : h->mycol;
      for (int i = 0; i < m; ++i) {
        const int w = odd ? i * h->q + h->mycol : h->myrow * h->q + i;
        char* base = h->fz_base[w];
        f.P[i] = reinterpret_cast<double2*>(base + (odd ? FL.po : FL.pe));
        f.out[i] = reinterpret_cast<double2*>(base + (odd ? FL.bw + (size_t)r.off * FL.ldb * es
                                                          : FL.cw + (size_t)r.off * FL.ldc * es));
        // one flag array per step parity: the two communicators of a rank progress independently,
        // so a peer already in step s+1 must not overwrite flags this rank still reads for step s
        f.flags[i] = reinterpret_cast<unsigned*>(base + FL.flags) +
                     (odd ? 0 : (size_t)FL.tiles_max * std::max(h->p, h->q));
        f.done[i] = reinterpret_cast<unsigned long long*>(base + FL.done);
      }
      f.ldP = odd ? FL.ldpo : FL.ldpe;
      f.slot = (long long)f.ldP * h->n_max;
      f.done_target = h->fused_delivered;
      f.owner_beta = s > 1 ? 1 : 0;
      f.err = h->d_err;
      static const bool plain = getenv("CHASE_FUSED_PLAIN") != nullptr;
      f.plain = (m == 1 && plain) ? 1 : 0;
      f.tile_ctr = reinterpret_cast<unsigned long long*>(h->fz_base[me_world] + FL.ctr);
      f.ctr_base = 0;                        // local counter, reset per launch (stream-ordered;
      //                                        CTAs grab ahead, so grabs per launch vary)
      g.use_beta = 0;                        // the tile owner adds beta * old after the sum
      const bool cplx = h->dt == CHASE_C128;
      const int BMf = cplx ? ZG_BM : DG_BM, BNf = cplx ? ZG_BN : DG_BN;
      const int BNn = cplx ? ZG_BN_NARROW : DG_BN_NARROW;
      // ragged width: the N mod BN remainder columns as a second, narrow-tile fused launch when
      // that pads less (own tile-index and staging-column ranges, so the two launches of the step
      // never share a flag or a slot)
      static const bool no_narrow = getenv("CHASE_NO_NARROW") != nullptr;
      const int rem = g.N % BNf;
      const bool split_w = !no_narrow && rem != 0 && (rem + BNn - 1) / BNn * BNn < BNf;
      const int Nmain = split_w ? g.N - rem : g.N;
      const int cat = odd ? CAT_HEMM_ODD : CAT_HEMM_EVEN;
      ProfScope ps(h, cat, 0);
      // wave tail (fused_tail.cuh): when the step's tiles leave the persistent grid's last round
      // partly idle, the fused kernel runs the first T_main tiles and the last T_tail tiles are
      // split over K and reduced through the tail slots (slot pair per step parity, alternating)
      static const bool no_tail = getenv("CHASE_FUSED_NO_TAIL") != nullptr;
      const int G = h->sm_budget > 0 ? std::min(h->sm_budget, h->num_sms) : h->num_sms;
      // the plan must be identical on every member (they process the same tile sets): K = the
      // member's local rows differs by up to a block across members, so plan with the largest
      const int Kplan = (int)(odd ? FL.ldc : FL.ldb);
      const int KTf = (Kplan + (cplx ? ZG_BK : DG_BKT) - 1) / (cplx ? ZG_BK : DG_BKT);
      const int tslot = (odd ? 0 : 2) + (int)(h->fused_tail_k[odd ? 0 : 1]++ & 1u);
      FusedTailArgs tbase{};
      tbase.m = m;
      tbase.me = f.me;
      tbase.M = g.M;
      tbase.ldo = g.ldo;
      tbase.ldx = g.ldx;
      tbase.alpha = g.alpha;
      tbase.beta = g.beta;
      tbase.c = g.c;
      tbase.owner_beta = f.owner_beta;
      tbase.band_lo = g.band_lo;
      tbase.band_hi = g.band_hi;
      tbase.band_shift = g.band_shift;
      tbase.band_map = g.band_map;
      tbase.err = h->d_err;
      tbase.sub = (long long)FUSED_TAIL_TILES * 128 * 128 * 8 / es;   // elements per sub-slot
      for (int i = 0; i < m; ++i) {
        const int w = odd ? i * h->q + h->mycol : h->myrow * h->q + i;
        char* base = h->fz_base[w];
        tbase.tp[i] = base + FL.tailp + (size_t)tslot * std::max(h->p, h->q) * FUSED_TAIL_TILES * 128 * 128 * 8;
        tbase.tflag[i] = reinterpret_cast<unsigned*>(base + FL.tflags) + (size_t)tslot * FUSED_MAX_MEMBERS;
      }
      FusedTailArgs tpend[2];
      void* tout[2] = {nullptr, nullptr};
      bool tnar[2] = {false, false};
      int npend = 0, slot_used = 0;
      int tile_base = 0;
      for (int part = 0; part < (split_w ? 2 : 1); ++part) {
        GemmReq gp = g;
        const bool nar = part == 1;
        FusedArgs fp = f;
        if (nar) {
          gp.N = rem;
          gp.tX = g.tX_narrow;
          gp.x_n0 = g.x_n0 + Nmain;
          gp.xin = static_cast<const char*>(g.xin) + (size_t)Nmain * g.ldx * es;
          for (int i = 0; i < m; ++i) fp.out[i] = reinterpret_cast<double2*>(
              reinterpret_cast<char*>(f.out[i]) + (size_t)Nmain * g.ldo * es);
          fp.col_base = Nmain;
        } else {
          gp.N = Nmain;
        }
        if (gp.N <= 0) continue;
        const int T = ((gp.M + BMf - 1) / BMf) * ((gp.N + (nar ? BNn : BNf) - 1) / (nar ? BNn : BNf));
        int tS = 1, tail = 0;
        if (!no_tail && !f.plain && T >= G)
          plan_tail(T, KTf, G, FUSED_TAIL_TILES - slot_used, &tS, &tail);
        const int tmain = T - tail;
        fp.tile_base = tile_base;
        fp.tiles = tail > 0 ? tmain : 0;
        if (tmain > 0) {
          fp.ep = ++h->fused_ep;
          CUDA_TRY(cudaMemsetAsync(f.tile_ctr, 0, sizeof(unsigned long long), h->stream));
          STATUS_TRY(launch_zgemm_fused(h, gp.conj, *gp.tA, *gp.tX, gp, fp, tmain, nar));
          h->launches[cat] += 1;
          h->fused_delivered += (unsigned long long)tmain;
        } else if (tail > 0) {
          // no fused kernel to wait for the previous step's deliveries: the split-K tail reads them
          fused_wait_kernel<<<1, 1, 0, h->stream>>>(f.done[f.me], h->fused_delivered, h->d_err);
          CUDA_TRY(cudaGetLastError());
          h->launches[cat] += 1;
        }
        tile_base += T;
        if (tail == 0) continue;
        GemmReq t = gp;
        t.narrow = nar ? 1 : 0;
        t.tX_narrow = nullptr;
        t.k_split = tS;
        t.tail_tiles = tail;
        t.tile_offset = tmain;
        t.out = h->tailws;
        t.ldo = BMf;
        t.alpha = 1.0; t.beta = 0.0; t.c = 0.0; t.use_beta = 0;
        t.band_lo = t.band_hi = 0; t.band_shift = 0; t.band_map = nullptr;
        STATUS_TRY(run_gemm(h, t));
        FusedTailArgs ta = tbase;
        ta.S = tS;
        ta.tail_tiles = tail;
        ta.tile_offset = tmain;
        ta.slot_off = slot_used;
        ta.N = gp.N;
        if (cplx && !nar)
          fused_tail_publish_kernel<double2, ZG_BM, ZG_BN, ZG_GROUP_M><<<tail, 256, 0, h->stream>>>(
              reinterpret_cast<const double2*>(h->tailws), static_cast<const double2*>(gp.xin), ta);
        else if (cplx)
          fused_tail_publish_kernel<double2, ZG_BM, ZG_BN_NARROW, ZG_GROUP_M><<<tail, 256, 0, h->stream>>>(
              reinterpret_cast<const double2*>(h->tailws), static_cast<const double2*>(gp.xin), ta);
        else if (!nar)
          fused_tail_publish_kernel<double, DG_BM, DG_BN, DG_GROUP_M><<<tail, 256, 0, h->stream>>>(
              reinterpret_cast<const double*>(h->tailws), static_cast<const double*>(gp.xin), ta);
        else
          fused_tail_publish_kernel<double, DG_BM, DG_BN_NARROW, DG_GROUP_M><<<tail, 256, 0, h->stream>>>(
              reinterpret_cast<const double*>(h->tailws), static_cast<const double*>(gp.xin), ta);
        CUDA_TRY(cudaGetLastError());
        h->launches[cat] += 2;                 // split-K copies + publish
        tpend[npend] = ta;
        tout[npend] = fp.out[f.me];
        tnar[npend] = nar;
        ++npend;
        slot_used += tail;
      }
      if (npend > 0) {
        tbase.ep = ++h->fused_ep;
        fused_tail_sync_kernel<<<1, 1, 0, h->stream>>>(tbase);
        CUDA_TRY(cudaGetLastError());
        h->launches[cat] += 1 + npend;
        for (int i = 0; i < npend; ++i) {
          FusedTailArgs ta = tpend[i];
          const int nt = ta.tail_tiles;
          if (cplx && !tnar[i])
            fused_tail_reduce_kernel<double2, ZG_BM, ZG_BN, ZG_GROUP_M><<<nt, 256, 0, h->stream>>>(
                static_cast<double2*>(tout[i]), ta);
          else if (cplx)
            fused_tail_reduce_kernel<double2, ZG_BM, ZG_BN_NARROW, ZG_GROUP_M><<<nt, 256, 0, h->stream>>>(
                static_cast<double2*>(tout[i]), ta);
          else if (!tnar[i])
            fused_tail_reduce_kernel<double, DG_BM, DG_BN, DG_GROUP_M><<<nt, 256, 0, h->stream>>>(
                reinterpret_cast<double*>(tout[i]), ta);
          else
            fused_tail_reduce_kernel<double, DG_BM, DG_BN_NARROW, DG_GROUP_M><<<nt, 256, 0, h->stream>>>(
                reinterpret_cast<double*>(tout[i]), ta);
          CUDA_TRY(cudaGetLastError());
        }
      }
      continue;
    }
    if (fused) {
      // a local step reads what the previous fused step's owners delivered: wait for all of it
      const FusedLayout& L = FL;
      fused_wait_kernel<<<1, 1, 0, h->stream>>>(
          reinterpret_cast<const unsigned long long*>(h->fz_base[me_world] + L.done),
          h->fused_delivered, h->d_err);
      CUDA_TRY(cudaGetLastError());
    }
    {
      ProfScope ps(h, odd ? CAT_HEMM_ODD : CAT_HEMM_EVEN, 1);
      STATUS_TRY(run_gemm_tail(h, g));
    }
    if (fused) continue;                     // single-member communicator: nothing to reduce
    if (odd && h->p > 1) STATUS_TRY(allreduce(h, g.out, (size_t)ldb * r.k, h->ccomm));
    if (!odd && h->q > 1) {
      if (ldv == n_r)
        STATUS_TRY(allreduce(h, g.out, (size_t)n_r * r.k, h->rcomm));
      else
        STATUS_TRY(allreduce_cols(h, g.out, n_r, ldv, r.k, h->rcomm));
    }
  }
  if (fused) {
    // every tile of the last step delivered here, then the result leaves the symmetric buffer
    char* base = h->fz_base[me_world];
    fused_wait_kernel<<<1, 1, 0, h->stream>>>(reinterpret_cast<const unsigned long long*>(base + FL.done),
                                              h->fused_delivered, h->d_err);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpy2DAsync(V, ldv * es, Cbuf, ldc * es, n_r * es, ncols,
                               cudaMemcpyDeviceToDevice, h->stream));
    CUDA_TRY(cudaMemcpyAsync(h->h_info, h->d_err, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (*h->h_info != 0) {
      // the delivery counters no longer match h->fused_delivered on every member: the handle
      // refuses further fused calls until chase_set_fused_workspace re-zeroes them collectively
      fprintf(stderr, "[chase] fused filter: peer wait timed out\n");
      h->fused_broken = true;
      return CHASE_ECUDA;
    }
  }
  h->record = rec;
  h->last_matvecs = mv;
  if (stats) {
    stats->matvecs = mv;
    stats->steps = D;
  }
  return CHASE_OK;
}

// Diagnostics: this rank's partial of one filter step, no reduction (include/chase.h).
chase_status_t chase_filter_step(chase_handle_t h, const void* A_local, int64_t lda, const void* X,
                                 int64_t ldx, void* Y, int64_t ldy, int64_t k, int32_t odd,
                                 double alpha, double beta, double c, int32_t use_beta) {
  if (!h || !A_local || !X || !Y) return CHASE_EINVAL;
  if (k < 1 || k > h->n_max || lda < h->n_r) return CHASE_EINVAL;
  const int64_t rows_in = odd ? h->n_r : h->n_c, rows_out = odd ? h->n_c : h->n_r;
  if (ldx < rows_in || ldy < rows_out) return CHASE_EINVAL;
  if (!std::isfinite(alpha) || !std::isfinite(beta) || !std::isfinite(c)) return CHASE_EINVAL;
  if (!h->ws) return CHASE_ESTATE;
  const size_t es = esize_of(h->dt);
  if ((reinterpret_cast<uintptr_t>(A_local) & 15) || (reinterpret_cast<uintptr_t>(X) & 15) ||
      (reinterpret_cast<uintptr_t>(Y) & 15))
    return CHASE_EINVAL;
  if (((size_t)lda * es) % 16 || ((size_t)ldx * es) % 16) return CHASE_EINVAL;
  // the band of this rank (reading #6), exactly as build_schedule records it
  std::vector<chase_step_record_t> rec;
  int64_t mv;
  const int32_t degs2[1] = {2};
  build_schedule(Geom{h->n_r, h->n_c, h->r0, h->c0, h->myrow, h->mycol, h->nb}, 1, degs2, &rec, &mv);
  const chase_step_record_t& r = rec[odd ? 0 : 1];
  CUtensorMap tA, tX, tXn;
  int a3d = 0;
  STATUS_TRY(make_role_map(h, &tA, A_local, h->n_r, h->n_c, lda, odd ? ROLE_A_TRANS : ROLE_A_NOTRANS,
                           odd ? nullptr : &a3d));
  STATUS_TRY(make_role_map(h, &tX, X, rows_in, k, ldx, ROLE_X));
  STATUS_TRY(make_role_map(h, &tXn, X, rows_in, k, ldx, ROLE_X_NARROW));
  GemmReq g{};
  g.conj = odd != 0;
  g.tA = &tA; g.tX = &tX; g.tX_narrow = &tXn; g.a3d = a3d;
  g.M = (int)rows_out; g.N = (int)k; g.K = (int)rows_in;
  g.out = Y; g.ldo = ldy;
  g.xin = X; g.ldx = ldx;
  g.alpha = alpha; g.beta = beta; g.c = c;
  g.use_beta = use_beta ? 1 : 0;
  g.band_lo = r.band_lo; g.band_hi = r.band_hi;
  g.band_shift = odd ? (int)(h->c0 - h->r0) : (int)(h->r0 - h->c0);
  g.band_map = h->nb > 0 ? (odd ? h->d_band_odd : h->d_band_even) : nullptr;
  ProfScope ps(h, odd ? CAT_HEMM_ODD : CAT_HEMM_EVEN, 1);
  return run_gemm_tail(h, g);
}

}  // extern "C"

// ==================================================================== CholeskyQR (Alg.3/4)
namespace {

// diagonal block kb: R_kk and R_kk^{-1} (into Rinv[:, kb:kb+64], ld 64)
template <typename T>
void potrf_diag(chase_handle_s* h, char* G, int64_t ldg, int kb, int nb) {
  potrf_diag_kernel<T><<<1, POTRF_DIAG_THREADS, diag_smem<T>(), h->stream>>>(
      reinterpret_cast<T*>(G), ldg, kb, nb, h->d_info, reinterpret_cast<T*>(h->Rinv) + (size_t)kb * QR_NB);
  h->launches[CAT_POTRF]++;
}

struct QrMaps {
  CUtensorMap vA_t, vA_nt, vX, gA_t, gX, wA_nt, rinvX, rinvA_t;
  CUtensorMap gA_nt, rfA_nt, rfX, tmpX;      // TRSM through R^{-1} (recursive doubling)
  int v_a3d = 0, w_a3d = 0;
};

// Split-K factor of the Gram GEMM: the upper-triangle tiles of an n x n output are few (C2:
// ~600 tiles = 4.05 waves on 148 SMs); S K-slices of them fill the waves.  S minimises the
// modelled waves (in units of a full-K tile), with K/S >= 1024 and the S partial n x n matrices
// fitting in the W workspace.
static int gram_split(const chase_handle_s* h, int n, int64_t K) {
  static const bool off = getenv("CHASE_NO_GRAM_SPLIT") != nullptr;   // A/B switch
  if (off) return 1;
  const bool cplx = h->dt == CHASE_C128;
  const int BM = cplx ? ZG_BM : DG_BM, BN = cplx ? ZG_BN : DG_BN;
  const int n_tiles = (n + BN - 1) / BN, m_tiles = (n + BM - 1) / BM;
  int64_t up = 0;
  for (int j = 0; j < n_tiles; ++j) up += std::min<int64_t>(m_tiles, (int64_t)(j * BN + BN - 1) / BM + 1);
  const int64_t wcap = (std::max(h->n_r, h->n_c) + 2) * h->n_max;           // W elements
  const int64_t mat = pad_ld(n) * (int64_t)n;
  int best = 1;
  double best_w = (double)((up + h->num_sms - 1) / h->num_sms);
  for (int S = 2; S <= 8; ++S) {
    if (K / S < 1024 || S * mat > wcap) break;
    const double w = (double)((up * S + h->num_sms - 1) / h->num_sms) / S;
    if (w < best_w - 0.02) {
      best_w = w;
      best = S;
    }
  }
  return best;
}

// One Gram/POTRF/TRSM round; returns CHASE_ECHOL with *info set when POTRF fails (V untouched).
chase_status_t cholqr_pass(chase_handle_s* h, void* V, int64_t ldv, int n, bool shifted,
                           const QrMaps& mp, int* info) {
  const size_t es = esize_of(h->dt);
  const int64_t n_r = h->n_r;
  char* G = static_cast<char*>(h->Gws);
  char* Vc = static_cast<char*>(V);
  const int64_t ldg = pad_ld(n);
  // Gram G = V^H V (upper tiles), Alg.3 l.3; split over K into partials in W when that fills
  // the waves better, then summed in fixed order (deterministic)
  {
    const int S = gram_split(h, n, n_r);
    GemmReq g{};
    g.conj = true; g.tA = &mp.vA_t; g.tX = &mp.vX;
    g.M = n; g.N = n; g.K = (int)n_r;
    g.out = S > 1 ? h->Wws : G; g.ldo = ldg; g.xin = nullptr; g.ldx = 0;
    g.alpha = 1.0; g.beta = 0.0; g.c = 0.0; g.use_beta = 0;
    g.band_lo = g.band_hi = 0; g.band_shift = 0; g.upper_only = 1; g.abort_flag = nullptr;
    g.k_split = S; g.split_ld = (int64_t)ldg * n;
    ProfScope ps(h, CAT_GRAM, S > 1 ? 2 : 1);
    STATUS_TRY(run_gemm(h, g));
    if (S > 1) {
      const dim3 grid((unsigned)((n + 255) / 256), (unsigned)n);
      if (h->dt == CHASE_C128)
        hh_splitsum_kernel<double2><<<grid, 256, 0, h->stream>>>(
            static_cast<const double2*>(h->Wws), (long long)ldg * n, S, n, (int)ldg,
            reinterpret_cast<double2*>(G), (int)ldg);
      else
        hh_splitsum_kernel<double><<<grid, 256, 0, h->stream>>>(
            static_cast<const double*>(h->Wws), (long long)ldg * n, S, n, (int)ldg,
            reinterpret_cast<double*>(G), (int)ldg);
      CUDA_TRY(cudaGetLastError());
    }
  }
  // Alg.3 l.4 AllReduce over the column communicator
  if (h->p > 1) STATUS_TRY(allreduce(h, G, (size_t)ldg * n, h->ccomm));
  if (shifted) {
    ProfScope ps(h, CAT_OTHER, 1);
    if (h->dt == CHASE_C128)
      shift_kernel<double2><<<1, 256, 0, h->stream>>>(reinterpret_cast<double2*>(G), ldg, n, h->N, h->d_shift);
    else
      shift_kernel<double><<<1, 256, 0, h->stream>>>(reinterpret_cast<double*>(G), ldg, n, h->N, h->d_shift);
    CUDA_TRY(cudaGetLastError());
  }
  // POTRF, blocked right-looking, Alg.3 l.5
  {
    ProfScope ps(h, CAT_POTRF, 0);
    CUDA_TRY(cudaMemsetAsync(h->d_info, 0, sizeof(int), h->stream));
    for (int kb = 0; kb < n; kb += QR_NB) {
      const int nb = std::min(QR_NB, n - kb);
      const int rest = n - kb - nb;
      if (h->dt == CHASE_C128)
        potrf_diag<double2>(h, G, ldg, kb, nb);
      else
        potrf_diag<double>(h, G, ldg, kb, nb);
      CUDA_TRY(cudaGetLastError());
      if (rest > 0) {
        // block row R[kb, kb+nb:] = R_kk^{-H} G[kb, kb+nb:] on the tensor cores, in place (one
        // m-tile: every CTA reads only the columns it writes, all its k-tiles before its epilogue)
        GemmReq g{};
        g.conj = true; g.tA = &mp.rinvA_t; g.tX = &mp.gX;
        g.M = nb; g.N = rest; g.K = nb;
        g.a_d0 = 0; g.a_d1 = kb; g.x_k0 = kb; g.x_n0 = kb + nb;
        g.out = G + ((size_t)kb + (size_t)(kb + nb) * ldg) * es; g.ldo = ldg;
        g.alpha = 1.0; g.abort_flag = h->d_info;
        STATUS_TRY(run_gemm(h, g));
        h->launches[CAT_POTRF]++;
      }
      if (rest > 0) {
        // trailing HERK: G[j, l] -= sum_a conj(R[a, j]) R[a, l], a in the panel, j <= l
        GemmReq g{};
        g.conj = true; g.tA = &mp.gA_t; g.tX = &mp.gX;
        g.M = rest; g.N = rest; g.K = nb;
        g.a_d0 = kb; g.a_d1 = kb + nb; g.x_k0 = kb; g.x_n0 = kb + nb;
        g.out = G + ((size_t)(kb + nb) + (size_t)(kb + nb) * ldg) * es; g.ldo = ldg;
        g.alpha = -1.0; g.beta = 1.0; g.c = 0.0; g.use_beta = 1;
        g.band_lo = g.band_hi = 0; g.upper_only = 1; g.abort_flag = h->d_info;
        STATUS_TRY(run_gemm(h, g));
        h->launches[CAT_POTRF]++;
      }
    }
    CUDA_TRY(cudaMemcpyAsync(h->h_info, h->d_info, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    if (shifted)
      CUDA_TRY(cudaMemcpyAsync(h->h_shift, h->d_shift, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  *info = *h->h_info;
  if (shifted) h->last_shift = *h->h_shift;
  if (*info != 0) return CHASE_ECHOL;
  // TRSM V <- V R^{-1}, Alg.3 l.6, as R^{-1} by recursive doubling + ONE GEMM:
  //   64x64 diagonal blocks inverted in smem (trtri_diag_kernel); then for b = 64, 128, ...:
  //   each pair of inverted b-blocks becomes a 2b-block, X12 = -R11^{-1} (R12 R22^{-1});
  //   W = V R^{-1} on the tensor cores with a triangular K range per output tile (tri_k, longest
  //   tiles first); W copied back into V.  The products X R^{-1} differ from a triangular solve
  //   by O(u kappa(R)^2) inside span(X) and O(u kappa(R)) across it -- within CholeskyQR's own
  //   u kappa^2 (Gram) loss, which the next pass removes (TRSM).
  static const bool blocked_trsm = getenv("CHASE_TRSM_BLOCKED") != nullptr;   // A/B switch
  if (!blocked_trsm) {
    ProfScope ps(h, CAT_TRSM, 0);
    const int64_t ldf = pad_ld(n), ldw = pad_ld(n_r);
    char* Rf = h->Rfws;
    char* Tmp = h->Rfws + align256((size_t)pad_ld(h->n_max) * h->n_max * es);
    char* W = static_cast<char*>(h->Wws);
    const int nblk = (n + TRTRI_NB - 1) / TRTRI_NB;
    CUDA_TRY(cudaMemsetAsync(Rf, 0, (size_t)ldf * n * es, h->stream));
    if (h->dt == CHASE_C128)
      trtri_diag_kernel<double2><<<nblk, TRTRI_NB, trtri_smem<double2>(), h->stream>>>(
          reinterpret_cast<const double2*>(G), ldg, n, reinterpret_cast<double2*>(Rf), ldf, 1);
    else
      trtri_diag_kernel<double><<<nblk, TRTRI_NB, trtri_smem<double>(), h->stream>>>(
          reinterpret_cast<const double*>(G), ldg, n, reinterpret_cast<double*>(Rf), ldf, 1);
    CUDA_TRY(cudaGetLastError());
    h->launches[CAT_TRSM]++;
    // level b: pairs p = 0..np-1 at i0 = 2 b p (block-diagonal, independent): the full pairs in
    // one batched launch per product, a trailing short pair (b2 < b) in its own
    for (int b = TRTRI_NB; b < n; b *= 2) {
      const int npairs = (n - b + 2 * b - 1) / (2 * b);       // pairs with i0 + b < n
      const int nfull = (n / (2 * b));                          // pairs with b2 == b
      for (int part = 0; part < 2; ++part) {
        const int p0 = part == 0 ? 0 : nfull, cnt = part == 0 ? nfull : npairs - nfull;
        if (cnt <= 0) continue;
        const int i0 = 2 * b * p0, j0 = i0 + b, b2 = std::min(i0 + 2 * b, n) - j0;
        const int st = 2 * b;
        GemmReq g{};                          // Tmp[i0:j0, j0:j0+b2] = R[i0:j0, j0:j0+b2] R22^{-1}
        g.conj = false; g.tA = &mp.gA_nt; g.tX = &mp.rfX;
        g.M = b; g.N = b2; g.K = b2;
        g.a_d0 = i0; g.a_d1 = j0; g.x_k0 = j0; g.x_n0 = j0;
        g.out = Tmp + ((size_t)i0 + (size_t)j0 * ldf) * es; g.ldo = ldf; g.alpha = 1.0;
        g.nbatch = cnt; g.bat_a = st; g.bat_x = st; g.bat_out = (int64_t)st * (1 + ldf);
        g.tri_k = 1;                          // R22^{-1} upper triangular: k < n0 + BN per tile
        STATUS_TRY(run_gemm(h, g));
        GemmReq g2{};                         // X12 = -R11^{-1} Tmp
        g2.conj = false; g2.tA = &mp.rfA_nt; g2.tX = &mp.tmpX;
        g2.M = b; g2.N = b2; g2.K = b;
        g2.a_d0 = i0; g2.a_d1 = i0; g2.x_k0 = i0; g2.x_n0 = j0;
        g2.out = Rf + ((size_t)i0 + (size_t)j0 * ldf) * es; g2.ldo = ldf; g2.alpha = -1.0;
        g2.nbatch = cnt; g2.bat_a = st; g2.bat_x = st; g2.bat_out = (int64_t)st * (1 + ldf);
        STATUS_TRY(run_gemm(h, g2));
        h->launches[CAT_TRSM] += 2;
      }
    }
    {
      GemmReq g{};                            // W = V R^{-1}
      g.conj = false; g.tA = &mp.vA_nt; g.tX = &mp.rfX; g.a3d = mp.v_a3d;
      g.M = (int)n_r; g.N = n; g.K = n; g.tri_k = 1;
      g.out = W; g.ldo = ldw; g.alpha = 1.0;
      STATUS_TRY(run_gemm(h, g));
      h->launches[CAT_TRSM]++;
    }
    CUDA_TRY(cudaMemcpy2DAsync(Vc, ldv * es, W, ldw * es, n_r * es, n, cudaMemcpyDeviceToDevice,
                               h->stream));
    return CHASE_OK;
  }
  // blocked variant (CHASE_TRSM_BLOCKED): right-looking with inverted 64x64 diagonal blocks.
  // Solved block columns go to W (W_k = V_k Rinv_kk), the trailing columns of V are updated
  // with V_rest -= W_k R[k, rest]; W is copied back into V at the end.
  {
    ProfScope ps(h, CAT_TRSM, 0);
    const int nblk = (n + TRTRI_NB - 1) / TRTRI_NB;
    char* W = static_cast<char*>(h->Wws);
    const int64_t ldw = pad_ld(n_r);
    if (h->dt == CHASE_C128)
      trtri_diag_kernel<double2><<<nblk, TRTRI_NB, trtri_smem<double2>(), h->stream>>>(
          reinterpret_cast<const double2*>(G), ldg, n, reinterpret_cast<double2*>(h->Rinv));
    else
      trtri_diag_kernel<double><<<nblk, TRTRI_NB, trtri_smem<double>(), h->stream>>>(
          reinterpret_cast<const double*>(G), ldg, n, reinterpret_cast<double*>(h->Rinv));
    CUDA_TRY(cudaGetLastError());
    h->launches[CAT_TRSM]++;
    // two-level blocking: 64-column diagonal solves inside 256-column panels, so the trailing
    // update of the rest of V runs with K = 256 (4x fewer read-modify-write passes over V)
#ifndef CHASE_TRSM_OUTER
#define CHASE_TRSM_OUTER 512
#endif
    constexpr int OUTER = CHASE_TRSM_OUTER;
    auto update = [&](int k0, int kn, int c0, int cn) -> chase_status_t {
      // V[:, c0:c0+cn] -= W[:, k0:k0+kn] R[k0:k0+kn, c0:c0+cn]
      GemmReq g{};
      g.conj = false; g.tA = &mp.wA_nt; g.tX = &mp.gX; g.a3d = mp.w_a3d;
      g.M = (int)n_r; g.N = cn; g.K = kn;
      g.a_d0 = 0; g.a_d1 = k0; g.x_k0 = k0; g.x_n0 = c0;
      g.out = Vc + (size_t)c0 * ldv * es; g.ldo = ldv;
      g.alpha = -1.0; g.beta = 1.0; g.c = 0.0; g.use_beta = 1;
      g.band_lo = g.band_hi = 0; g.upper_only = 0; g.abort_flag = nullptr;
      h->launches[CAT_TRSM]++;
      return run_gemm(h, g);
    };
    for (int ob = 0; ob < n; ob += OUTER) {
      const int onb = std::min(OUTER, n - ob);
      for (int kb = ob; kb < ob + onb; kb += TRTRI_NB) {
        const int nb = std::min(TRTRI_NB, ob + onb - kb);
        {   // W[:, kb:kb+nb] = V[:, kb:kb+nb] Rinv_kk
          GemmReq g{};
          g.conj = false; g.tA = &mp.vA_nt; g.tX = &mp.rinvX; g.a3d = mp.v_a3d;
          g.M = (int)n_r; g.N = nb; g.K = nb;
          g.a_d0 = 0; g.a_d1 = kb; g.x_k0 = 0; g.x_n0 = kb;
          g.out = W + (size_t)kb * ldw * es; g.ldo = ldw;
          g.alpha = 1.0; g.beta = 0.0; g.c = 0.0; g.use_beta = 0;
          g.band_lo = g.band_hi = 0; g.upper_only = 0; g.abort_flag = nullptr;
          STATUS_TRY(run_gemm(h, g));
          h->launches[CAT_TRSM]++;
        }
        const int inner_rest = ob + onb - kb - nb;
        if (inner_rest > 0) STATUS_TRY(update(kb, nb, kb + nb, inner_rest));
      }
      const int rest = n - ob - onb;
      if (rest > 0) STATUS_TRY(update(ob, onb, ob + onb, rest));
    }
    CUDA_TRY(cudaMemcpy2DAsync(Vc, ldv * es, W, ldw * es, n_r * es, n, cudaMemcpyDeviceToDevice,
                               h->stream));
  }
  return CHASE_OK;
}

bool g_qr_attr_done = false;

#include "hhqr.inc"
#include "heevd.inc"

}  // namespace

extern "C" {

chase_status_t chase_cholqr(chase_handle_t h, void* V, int64_t ldv, int64_t ncols,
                            double cond_est, chase_stats_t* stats, int32_t* info_out) {
  Nvtx nv_("chase_cholqr");
  if (!h || !V) return CHASE_EINVAL;
  if (ncols < 1 || ncols > h->n_max || ldv < h->n_r) return CHASE_EINVAL;
  if (((size_t)ldv * esize_of(h->dt)) % 16) return CHASE_EINVAL;   // TMA pitch
  if (!(cond_est >= 1.0)) return CHASE_EINVAL;   // also rejects NaN
  if (!h->ws || (h->virt && h->p > 1)) return CHASE_ESTATE;
  if (reinterpret_cast<uintptr_t>(V) & 15) return CHASE_EINVAL;
  if (!g_qr_attr_done) {
    CUDA_TRY(cudaFuncSetAttribute(trtri_diag_kernel<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, trtri_smem<double2>()));
    CUDA_TRY(cudaFuncSetAttribute(potrf_diag_kernel<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, diag_smem<double2>()));
    CUDA_TRY(cudaFuncSetAttribute(potrf_diag_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, diag_smem<double>()));
    CUDA_TRY(cudaFuncSetAttribute(trtri_diag_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, trtri_smem<double>()));
    g_qr_attr_done = true;
  }
  const int n = (int)ncols;
  if (spmd_check_enabled()) {
    SpmdHash hs;
    hs.add(ncols);
    hs.add(cond_est);
    hs.add(h->qr_mode);
    STATUS_TRY(spmd_verify(h, hs.v));
  }
  QrMaps mp;
  STATUS_TRY(make_role_map(h, &mp.vA_t, V, h->n_r, n, ldv, ROLE_A_TRANS));
  STATUS_TRY(make_role_map(h, &mp.vA_nt, V, h->n_r, n, ldv, ROLE_A_NOTRANS, &mp.v_a3d));
  STATUS_TRY(make_role_map(h, &mp.vX, V, h->n_r, n, ldv, ROLE_X));
  STATUS_TRY(make_role_map(h, &mp.gA_t, h->Gws, n, n, pad_ld(n), ROLE_A_TRANS));
  STATUS_TRY(make_role_map(h, &mp.gX, h->Gws, n, n, pad_ld(n), ROLE_X));
  STATUS_TRY(make_role_map(h, &mp.wA_nt, h->Wws, h->n_r, n, pad_ld(h->n_r), ROLE_A_NOTRANS, &mp.w_a3d));
  STATUS_TRY(make_role_map(h, &mp.rinvX, h->Rinv, TRTRI_NB, n, TRTRI_NB, ROLE_X));
  STATUS_TRY(make_role_map(h, &mp.rinvA_t, h->Rinv, TRTRI_NB, n, TRTRI_NB, ROLE_A_TRANS));
  {
    char* Rf = h->Rfws;
    char* Tmp = h->Rfws + align256((size_t)pad_ld(h->n_max) * h->n_max * esize_of(h->dt));
    STATUS_TRY(make_role_map(h, &mp.gA_nt, h->Gws, n, n, pad_ld(n), ROLE_A_NOTRANS));
    STATUS_TRY(make_role_map(h, &mp.rfA_nt, Rf, n, n, pad_ld(n), ROLE_A_NOTRANS));
    STATUS_TRY(make_role_map(h, &mp.rfX, Rf, n, n, pad_ld(n), ROLE_X));
    STATUS_TRY(make_role_map(h, &mp.tmpX, Tmp, n, n, pad_ld(n), ROLE_X));
  }

  // Alg.4: est > 1e8 -> shifted CholeskyQR2; est < 20 -> CholeskyQR; else CholeskyQR2
  int variant = cond_est > 1e8 ? CHASE_QR_SHIFTED : (cond_est < 20.0 ? CHASE_QR_CHOL1 : CHASE_QR_CHOL2);
  int info = 0, passes = 0;
  h->last_shift = 0.0;
  chase_status_t st = CHASE_OK;
  bool hh = h->qr_mode == 1;                     // HHQR in every call (Table 3)
  if (!hh && variant != CHASE_QR_SHIFTED) {
    const int rounds = variant == CHASE_QR_CHOL1 ? 1 : 2;
    for (int i = 0; i < rounds; ++i) {
      st = cholqr_pass(h, V, ldv, n, false, mp, &info);
      if (st != CHASE_OK) break;
      ++passes;
    }
    if (st == CHASE_ECHOL) {
      if (passes == 0) variant = CHASE_QR_SHIFTED;   // reading #14: escalate, V untouched
      else hh = true;                                // reading #33: HHQR on the current V
      st = CHASE_OK;
    }
  }
  if (!hh && variant == CHASE_QR_SHIFTED && st == CHASE_OK && passes == 0) {
    st = cholqr_pass(h, V, ldv, n, true, mp, &info);
    if (st == CHASE_OK) {
      ++passes;
      for (int i = 0; i < 2 && st == CHASE_OK; ++i) {
        st = cholqr_pass(h, V, ldv, n, false, mp, &info);
        if (st == CHASE_OK) ++passes;
      }
    }
    if (st == CHASE_ECHOL) {                        // Alg.4 l.8-9; reading #33
      hh = true;
      st = CHASE_OK;
    }
  }
  if (hh && st == CHASE_OK) {
    variant = CHASE_QR_HOUSEHOLDER;
    st = hhqr_run(h, V, ldv, n);
  }
  if (stats) {
    stats->qr_variant = variant;
    stats->qr_passes = passes;
    stats->shift = h->last_shift;
  }
  if (info_out) *info_out = info;
  return st;
}

chase_status_t chase_hhqr(chase_handle_t h, void* V, int64_t ldv, int64_t ncols) {
  Nvtx nv_("chase_hhqr");
  if (!h || !V) return CHASE_EINVAL;
  if (ncols < 1 || ncols > h->n_max || ldv < h->n_r) return CHASE_EINVAL;
  if (((size_t)ldv * esize_of(h->dt)) % 16) return CHASE_EINVAL;
  if (reinterpret_cast<uintptr_t>(V) & 15) return CHASE_EINVAL;
  if (!h->ws || (h->virt && h->p > 1)) return CHASE_ESTATE;
  return hhqr_run(h, V, ldv, (int)ncols);
}

chase_status_t chase_set_qr_mode(chase_handle_t h, int32_t mode) {
  if (!h || (mode != 0 && mode != 1)) return CHASE_EINVAL;
  h->qr_mode = mode;
  return CHASE_OK;
}

// Alg.2 l.16 / l.23 "B2 <- Bcast(C2, ccomm)": the rows [c0, c0+n_c) (block-cyclic: the column
// index set) of the C-layout block V, fetched from the rank(s) of the column communicator that
// own them (one Bcast per owning block; a square grid needs one).  *y2 / *ldy2 point
// to the B-layout copy (V itself on a 1x1 grid).
static chase_status_t redistribute_b2(chase_handle_s* h, const void* V, int64_t ldv, int n,
                                      const void** y2, int64_t* ldy2) {
  const size_t es = esize_of(h->dt), per = es / 8;
  const int64_t n_c = h->n_c, ldb = pad_ld(n_c);
  // l.23 B2 <- Bcast(C2, ccomm): rows [c0, c0+n_c) of V, from the rank(s) of this column
  // communicator that own them (one Bcast per owning block; a square grid needs one)
  const char* Vc = static_cast<const char*>(V);
  char* B2 = static_cast<char*>(h->B2ws);
  *y2 = B2;
  *ldy2 = ldb;
  if (h->p == 1 && h->q == 1) {
    *y2 = V;                                          // C- and B-layout coincide on a 1x1 grid
    *ldy2 = ldv;
  } else if (h->nb > 0) {
    // block-cyclic: the owner gathers its rows of my column set, Bcast, scatter into B2
    ProfScope ps(h, CAT_ALLREDUCE, 0);
    char* stage = static_cast<char*>(h->Wws);
    for (int i2 = 0; i2 < h->p; ++i2) {
      const int64_t a = h->b2_seg[i2], cnt = h->b2_seg[i2 + 1] - a;
      if (cnt == 0) continue;
      const dim3 grid((unsigned)((cnt + 255) / 256), (unsigned)n);
      if (h->myrow == i2) {
        if (h->dt == CHASE_C128)
          gather_rows_kernel<double2><<<grid, 256, 0, h->stream>>>(
              reinterpret_cast<const double2*>(V), ldv, h->d_b2_src + a, (int)cnt,
              reinterpret_cast<double2*>(stage));
        else
          gather_rows_kernel<double><<<grid, 256, 0, h->stream>>>(
              reinterpret_cast<const double*>(V), ldv, h->d_b2_src + a, (int)cnt,
              reinterpret_cast<double*>(stage));
        CUDA_TRY(cudaGetLastError());
      }
      if (h->p > 1)
        NCCL_TRY(ncclBroadcast(stage, stage, (size_t)cnt * n * per, ncclDouble, i2, h->ccomm, h->stream));
      if (h->dt == CHASE_C128)
        scatter_rows_kernel<double2><<<grid, 256, 0, h->stream>>>(
            reinterpret_cast<const double2*>(stage), h->d_b2_dst + a, (int)cnt,
            reinterpret_cast<double2*>(B2), ldb);
      else
        scatter_rows_kernel<double><<<grid, 256, 0, h->stream>>>(
            reinterpret_cast<const double*>(stage), h->d_b2_dst + a, (int)cnt,
            reinterpret_cast<double*>(B2), ldb);
      CUDA_TRY(cudaGetLastError());
    }
  } else {
    ProfScope ps(h, CAT_ALLREDUCE, 0);
    char* stage = static_cast<char*>(h->Wws);
    for (int i2 = 0; i2 < h->p; ++i2) {
      int64_t nr2, r02;
      block_part(h->N, h->p, i2, &nr2, &r02);
      const int64_t lo = std::max(h->c0, r02), hi = std::min(h->c0 + n_c, r02 + nr2);
      if (lo >= hi) continue;
      const int64_t rows = hi - lo;
      if (h->myrow == i2)
        CUDA_TRY(cudaMemcpy2DAsync(stage, rows * es, Vc + (size_t)(lo - h->r0) * es, ldv * es,
                                   rows * es, n, cudaMemcpyDeviceToDevice, h->stream));
      if (h->p > 1)
        NCCL_TRY(ncclBroadcast(stage, stage, (size_t)rows * n * per, ncclDouble, i2, h->ccomm,
                               h->stream));
      CUDA_TRY(cudaMemcpy2DAsync(B2 + (size_t)(lo - h->c0) * es, ldb * es, stage, rows * es,
                                 rows * es, n, cudaMemcpyDeviceToDevice, h->stream));
    }
  }
  return CHASE_OK;
}

// Alg.2 l.23-28: residual norms ||H v_j - lambda_j v_j|| of Ritz pairs.
chase_status_t chase_residuals(chase_handle_t h, const void* A_local, int64_t lda, const void* V,
                               int64_t ldv, int64_t ncols, const double* ritz, double* resid) {
  Nvtx nv_("chase_residuals");
  if (!h || !A_local || !V || !ritz || !resid) return CHASE_EINVAL;
  if (ncols < 1 || ncols > h->n_max || lda < h->n_r || ldv < h->n_r) return CHASE_EINVAL;
  for (int64_t j = 0; j < ncols; ++j)
    if (!std::isfinite(ritz[j])) return CHASE_EINVAL;
  if (!h->ws || (h->virt && h->p * h->q > 1)) return CHASE_ESTATE;
  const size_t es = esize_of(h->dt), per = es / 8;
  if ((reinterpret_cast<uintptr_t>(A_local) & 15) || (reinterpret_cast<uintptr_t>(V) & 15))
    return CHASE_EINVAL;
  if (((size_t)lda * es) % 16 || ((size_t)ldv * es) % 16) return CHASE_EINVAL;
  const int64_t n_r = h->n_r, n_c = h->n_c, ldb = pad_ld(n_c);
  const int n = (int)ncols;
  CUDA_TRY(cudaMemcpyAsync(h->d_ritz, ritz, ncols * sizeof(double), cudaMemcpyHostToDevice, h->stream));

  // l.23 B2 <- Bcast(C2, ccomm)
  const void* y2 = nullptr;
  int64_t ldy2 = 0;
  STATUS_TRY(redistribute_b2(h, V, ldv, n, &y2, &ldy2));
  // l.24-25 B <- H C - ritzv B2: the odd-step HEMM with the shift term fused in the epilogue of
  // the first rank of the column communicator (linear, so it commutes with the AllReduce)
  CUtensorMap tA_t, tC;
  STATUS_TRY(make_role_map(h, &tA_t, A_local, n_r, n_c, lda, ROLE_A_TRANS));
  STATUS_TRY(make_role_map(h, &tC, V, n_r, n, ldv, ROLE_X));
  char* Bc = static_cast<char*>(h->Bws);
  {
    GemmReq g{};
    g.conj = true; g.tA = &tA_t; g.tX = &tC;
    g.M = (int)n_c; g.N = n; g.K = (int)n_r;
    g.out = Bc; g.ldo = ldb;
    g.alpha = 1.0; g.beta = 0.0; g.c = 0.0; g.use_beta = 0;
    g.band_lo = g.band_hi = 0;
    g.col_shift = h->myrow == 0 ? h->d_ritz : nullptr;
    g.y2 = y2; g.ldy2 = ldy2;
    ProfScope ps(h, CAT_HEMM_ODD, 1);
    STATUS_TRY(run_gemm(h, g));
  }
  if (h->p > 1) STATUS_TRY(allreduce(h, Bc, (size_t)ldb * n, h->ccomm));
  // l.26 squared column norms of the local rows, l.27 AllReduce over rcomm, l.28 sqrt
  {
    ProfScope ps(h, CAT_OTHER, 2);
    if (h->dt == CHASE_C128)
      colnorm2_kernel<double2><<<n, 256, 0, h->stream>>>(reinterpret_cast<const double2*>(Bc), ldb, (int)n_c, h->d_nrm);
    else
      colnorm2_kernel<double><<<n, 256, 0, h->stream>>>(reinterpret_cast<const double*>(Bc), ldb, (int)n_c, h->d_nrm);
    CUDA_TRY(cudaGetLastError());
  }
  if (h->q > 1) {
    ProfScope ps(h, CAT_ALLREDUCE, 0);
    NCCL_TRY(ncclAllReduce(h->d_nrm, h->d_nrm, n, ncclDouble, ncclSum, h->rcomm, h->stream));
  }
  sqrt_kernel<<<(n + 255) / 256, 256, 0, h->stream>>>(h->d_nrm, n);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(resid, h->d_nrm, ncols * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return CHASE_OK;
}

// Alg.2 l.16-22: Rayleigh-Ritz on the orthonormal C-layout block V.
chase_status_t chase_rayleigh_ritz(chase_handle_t h, const void* A_local, int64_t lda, void* V,
                                   int64_t ldv, int64_t ncols, double* ritz, int32_t* sweeps_out) {
  Nvtx nv_("chase_rayleigh_ritz");
  if (!h || !A_local || !V || !ritz) return CHASE_EINVAL;
  if (ncols < 1 || ncols > h->n_max || lda < h->n_r || ldv < h->n_r) return CHASE_EINVAL;
  if (!h->ws || (h->virt && h->p * h->q > 1)) return CHASE_ESTATE;
  const size_t es = esize_of(h->dt);
  if ((reinterpret_cast<uintptr_t>(A_local) & 15) || (reinterpret_cast<uintptr_t>(V) & 15))
    return CHASE_EINVAL;
  if (((size_t)lda * es) % 16 || ((size_t)ldv * es) % 16) return CHASE_EINVAL;
  static bool attr = false;
  if (!attr) {
    CUDA_TRY(cudaFuncSetAttribute(jacobi_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, JAC_SMEM));
    attr = true;
  }
  const int n = (int)ncols;
  const int64_t n_r = h->n_r, n_c = h->n_c, ldb = pad_ld(n_c);
  const bool cplx = h->dt == CHASE_C128;

  // l.16 B2 <- Bcast(C2, ccomm)
  const void* y2 = nullptr;
  int64_t ldy2 = 0;
  STATUS_TRY(redistribute_b2(h, V, ldv, n, &y2, &ldy2));
  // l.17 B <- H C (the odd-step HEMM, no shift), AllReduce over ccomm
  CUtensorMap tA_t, tC, tB2, tB;
  STATUS_TRY(make_role_map(h, &tA_t, A_local, n_r, n_c, lda, ROLE_A_TRANS));
  STATUS_TRY(make_role_map(h, &tC, V, n_r, n, ldv, ROLE_X));
  char* Bc = static_cast<char*>(h->Bws);
  {
    GemmReq g{};
    g.conj = true; g.tA = &tA_t; g.tX = &tC;
    g.M = (int)n_c; g.N = n; g.K = (int)n_r;
    g.out = Bc; g.ldo = ldb; g.alpha = 1.0;
    ProfScope ps(h, CAT_HEMM_ODD, 1);
    STATUS_TRY(run_gemm(h, g));
  }
  if (h->p > 1) STATUS_TRY(allreduce(h, Bc, (size_t)ldb * n, h->ccomm));
  // l.18-19 A <- B2^H B, AllReduce over rcomm
  const int64_t np = eig_np(n), L = np / 32;
  char* E = h->eigws;
  const size_t mat = align256((size_t)np * np * 16);
  double2* Abuf[2] = {reinterpret_cast<double2*>(E), reinterpret_cast<double2*>(E + mat)};
  double2* Ybuf[2] = {reinterpret_cast<double2*>(E + 2 * mat), reinterpret_cast<double2*>(E + 3 * mat)};
  double2* Ubd = reinterpret_cast<double2*>(E + 4 * mat);
  char* tail = E + 5 * mat;
  double* d_w = reinterpret_cast<double*>(tail);
  tail += align256(np * sizeof(double));
  int* d_order = reinterpret_cast<int*>(tail);
  tail += align256(np * sizeof(int));
  int* d_perm = reinterpret_cast<int*>(tail);
  tail += align256((size_t)(L + 1) * L * sizeof(int));
  double* d_part = reinterpret_cast<double*>(tail);
  double* d_off = d_part + 2 * JAC_RED_BLOCKS;
  tail += align256(2 * JAC_RED_BLOCKS * sizeof(double) + 2 * sizeof(double));
  double2* bt_tmp = reinterpret_cast<double2*>(tail);      // tridiagonal back-transform products
  STATUS_TRY(make_role_map(h, &tB2, y2, n_c, n, ldy2, ROLE_A_TRANS));
  STATUS_TRY(make_role_map(h, &tB, Bc, n_c, n, ldb, ROLE_X));
  const int64_t ldq = pad_ld(n);                       // real quotient / sorted Y in the G region
  {
    GemmReq g{};
    g.conj = true; g.tA = &tB2; g.tX = &tB;
    g.M = n; g.N = n; g.K = (int)n_c;
    g.out = cplx ? static_cast<void*>(Abuf[0]) : h->Gws;
    g.ldo = cplx ? np : ldq; g.alpha = 1.0;
    ProfScope ps(h, CAT_GRAM, 1);
    STATUS_TRY(run_gemm(h, g));
  }
  if (h->q > 1)
    STATUS_TRY(allreduce(h, cplx ? static_cast<void*>(Abuf[0]) : h->Gws, (size_t)(cplx ? np : ldq) * n, h->rcomm));
  const unsigned TB = 256;
  const unsigned g2 = (unsigned)((np * np + TB - 1) / TB);
  if (!cplx)
    real_to_complex_kernel<<<(unsigned)(((int64_t)n * n + TB - 1) / TB), TB, 0, h->stream>>>(
        static_cast<const double*>(h->Gws), ldq, Abuf[0], np, n);
  // l.20 HEEVD.  Default: Householder tridiagonalisation + divide and conquer + back-transform
  // (tridiag.cuh / heevd.inc); CHASE_RR_JACOBI=1: the parallel block-Jacobi solver below.
  static const bool use_jacobi = getenv("CHASE_RR_JACOBI") != nullptr;
  if (!use_jacobi) {
    ProfScope ps_eig(h, CAT_OTHER, 0);
    HeevdScratch hs{Abuf[1], np, reinterpret_cast<double*>(Ybuf[1]), reinterpret_cast<double*>(Ubd),
                    (size_t)np * np * 2, bt_tmp};
    std::vector<double> w;
    int levels = 0;
    STATUS_TRY(heevd_tridiag(h, Abuf[0], np, n, Ybuf[0], np, w, hs, &levels));
    std::vector<int> cols(n);
    for (int k = 0; k < n; ++k) cols[k] = k;
    std::stable_sort(cols.begin(), cols.end(), [&](int a, int b) { return w[a] < w[b]; });
    for (int k = 0; k < n; ++k) ritz[k] = w[cols[k]];
    CUDA_TRY(cudaMemcpyAsync(d_order, cols.data(), n * sizeof(int), cudaMemcpyHostToDevice, h->stream));
    const unsigned gn2 = (unsigned)(((int64_t)n * n + 255) / 256);
    if (cplx)
      jacobi_gather_kernel<double2><<<gn2, 256, 0, h->stream>>>(Ybuf[0], np, n, d_order,
                                                                 static_cast<double2*>(h->Gws), ldq);
    else
      jacobi_gather_kernel<double><<<gn2, 256, 0, h->stream>>>(Ybuf[0], np, n, d_order,
                                                                static_cast<double*>(h->Gws), ldq);
    CUDA_TRY(cudaGetLastError());
    CUtensorMap tV2, tY2;
    int a3dV2 = 0;
    STATUS_TRY(make_role_map(h, &tV2, V, n_r, n, ldv, ROLE_A_NOTRANS, &a3dV2));
    STATUS_TRY(make_role_map(h, &tY2, h->Gws, n, n, ldq, ROLE_X));
    char* W = static_cast<char*>(h->Wws);
    const int64_t ldw = pad_ld(n_r);
    {
      GemmReq g{};
      g.conj = false; g.tA = &tV2; g.tX = &tY2; g.a3d = a3dV2;
      g.M = (int)n_r; g.N = n; g.K = n;
      g.out = W; g.ldo = ldw; g.alpha = 1.0;
      ProfScope ps(h, CAT_TRSM, 1);
      STATUS_TRY(run_gemm(h, g));
    }
    CUDA_TRY(cudaMemcpy2DAsync(V, ldv * es, W, ldw * es, n_r * es, n, cudaMemcpyDeviceToDevice, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (sweeps_out) *sweeps_out = levels;
    return CHASE_OK;
  }
  jacobi_init_kernel<<<g2, TB, 0, h->stream>>>(Abuf[0], Ybuf[0], Ubd, np, n, (int)np, 0.0);
  CUDA_TRY(cudaGetLastError());

  // l.20 HEEVD: parallel block Jacobi (eig.cuh).  Circle-method layouts over L blocks of 32:
  // round r pairs (L-1, r) and ((r+i) mod (L-1), (r-i) mod (L-1)); pair i sits at positions
  // (2i, 2i+1).  lay[r][pos] = logical block; perm tables map round r -> r+1 (and identity -> 0).
  const int R = (int)(L - 1);
  std::vector<std::vector<int>> lay(R, std::vector<int>(L));
  for (int r = 0; r < R; ++r)
    for (int i = 0; i < L / 2; ++i) {
      int a, b;
      if (i == 0) {
        a = (int)L - 1;
        b = r;
      } else {
        a = (r + i) % R;
        b = (r - i + R) % R;
      }
      lay[r][2 * i] = a;
      lay[r][2 * i + 1] = b;
    }
  // table t (t = 0..R-1): layout (t == 0 ? identity : lay[t-1]) -> lay[t]; table R: lay[R-1] -> lay[0]
  std::vector<int> perm((size_t)(R + 1) * L);
  for (int t = 0; t <= R; ++t) {
    std::vector<int> inv(L);
    const std::vector<int>* from = nullptr;
    std::vector<int> ident(L);
    for (int k = 0; k < L; ++k) ident[k] = k;
    from = (t == 0) ? &ident : &lay[t - 1];
    for (int k = 0; k < L; ++k) inv[(*from)[k]] = k;
    const std::vector<int>& to = lay[t == R ? 0 : t];
    for (int pos = 0; pos < L; ++pos) perm[(size_t)t * L + pos] = inv[to[pos]];
  }
  CUDA_TRY(cudaMemcpyAsync(d_perm, perm.data(), perm.size() * sizeof(int), cudaMemcpyHostToDevice, h->stream));
  CUtensorMap mAnt[2], mAx[2], mYnt[2], mUx, mUt;
  int a3dA[2], a3dY[2];
  for (int b = 0; b < 2; ++b) {
    STATUS_TRY(make_map(&mAx[b], Abuf[b], np, np, np, 16, 8, ZG_BN));
    a3dA[b] = 0;
    {
      chase_handle_s tmp = *h;   // dtype-independent complex maps
      tmp.dt = CHASE_C128;
      STATUS_TRY(make_role_map(&tmp, &mAnt[b], Abuf[b], np, np, np, ROLE_A_NOTRANS, &a3dA[b]));
      STATUS_TRY(make_role_map(&tmp, &mYnt[b], Ybuf[b], np, np, np, ROLE_A_NOTRANS, &a3dY[b]));
    }
  }
  STATUS_TRY(make_map(&mUx, Ubd, np, np, np, 16, 8, ZG_BN));
  STATUS_TRY(make_map(&mUt, Ubd, np, np, np, 16, 8, ZG_BM));
  int cur = 0;
  const dim3 gp((unsigned)g2);
  auto permute = [&](int t) -> chase_status_t {
    jacobi_perm_kernel<<<gp, TB, 0, h->stream>>>(Abuf[cur], Abuf[cur ^ 1], Ybuf[cur], Ybuf[cur ^ 1], np,
                                                 (int)np, d_perm + (size_t)t * L);
    CUDA_TRY(cudaGetLastError());
    cur ^= 1;
    return CHASE_OK;
  };
  auto zgemm_inplace = [&](bool conj, const CUtensorMap& tA, const CUtensorMap& tX, int a3d,
                           double2* out, int K, int diag) -> chase_status_t {
    ZGemmArgs a{};
    a.M = (int)np; a.N = (int)np; a.K = K;
    a.out = out; a.ldo = np; a.alpha = 1.0; a.a3d = a3d; a.diag_k = diag;
    return launch_zgemm(h, conj, tA, tX, a);
  };
  ProfScope ps_eig(h, CAT_OTHER, 0);
  if (L > 2) STATUS_TRY(permute(0));
  int sweeps = 0;
  const int max_sweeps = 40;
  // one inner sweep per pair visit: the outer block-Jacobi sweeps finish the job (measured
  // fastest: n = 3000 in 13 sweeps, 2.0 s vs 2.8 s with inner convergence)
  static const int inner_sweeps = getenv("CHASE_JAC_INNER") ? atoi(getenv("CHASE_JAC_INNER")) : 1;
  std::vector<double> off(2);
  bool converged = false;
  for (; sweeps < max_sweeps; ++sweeps) {
    for (int r = 0; r < (L > 2 ? R : 1); ++r) {
      jacobi_pair_kernel<<<(unsigned)(np / JAC_PW), JAC_THREADS, JAC_SMEM, h->stream>>>(Abuf[cur], np, Ubd, np, inner_sweeps);
      CUDA_TRY(cudaGetLastError());
      STATUS_TRY(zgemm_inplace(false, mAnt[cur], mUx, a3dA[cur], Abuf[cur], JAC_PW, 1));   // A U
      STATUS_TRY(zgemm_inplace(true, mUt, mAx[cur], 0, Abuf[cur], 2 * JAC_PW, 2));          // U^H A
      STATUS_TRY(zgemm_inplace(false, mYnt[cur], mUx, a3dY[cur], Ybuf[cur], JAC_PW, 1));   // Y U
      h->launches[CAT_OTHER] += 4;
      if (L > 2) STATUS_TRY(permute(r + 1));
    }
    jacobi_offnorm_kernel<<<JAC_RED_BLOCKS, 256, 0, h->stream>>>(Abuf[cur], np, (int)np, d_part);
    jacobi_offnorm_final<<<1, 32, 0, h->stream>>>(d_part, JAC_RED_BLOCKS, d_off);
    CUDA_TRY(cudaMemcpyAsync(off.data(), d_off, 2 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (!(off[0] > 1e-28 * off[1])) {
      ++sweeps;
      converged = true;
      break;
    }
  }
  // eigenvalues in physical order; physical column -> logical index; drop the padding; sort
  std::vector<double> w(np);
  jacobi_diag_kernel<<<(unsigned)((np + 255) / 256), 256, 0, h->stream>>>(Abuf[cur], np, (int)np, d_w);
  CUDA_TRY(cudaMemcpyAsync(w.data(), d_w, np * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  const std::vector<int>& fin = (L > 2) ? lay[0] : std::vector<int>{0, 1};
  std::vector<int> cols;
  for (int pos = 0; pos < np; ++pos) {
    const int logical = fin[pos / 32] * 32 + pos % 32;
    if (logical < n) cols.push_back(pos);
  }
  std::stable_sort(cols.begin(), cols.end(), [&](int a, int b) { return w[a] < w[b]; });
  for (int k = 0; k < n; ++k) ritz[k] = w[cols[k]];
  CUDA_TRY(cudaMemcpyAsync(d_order, cols.data(), n * sizeof(int), cudaMemcpyHostToDevice, h->stream));
  const unsigned gn = (unsigned)(((int64_t)n * n + 255) / 256);
  if (cplx)
    jacobi_gather_kernel<double2><<<gn, 256, 0, h->stream>>>(Ybuf[cur], np, n, d_order,
                                                              static_cast<double2*>(h->Gws), ldq);
  else
    jacobi_gather_kernel<double><<<gn, 256, 0, h->stream>>>(Ybuf[cur], np, n, d_order,
                                                             static_cast<double*>(h->Gws), ldq);
  CUDA_TRY(cudaGetLastError());
  // l.21 C <- C2 A (the eigenvectors), into W then back into V (l.22 C2 <- C is the caller's)
  CUtensorMap tV, tY;
  int a3dV = 0;
  STATUS_TRY(make_role_map(h, &tV, V, n_r, n, ldv, ROLE_A_NOTRANS, &a3dV));
  STATUS_TRY(make_role_map(h, &tY, h->Gws, n, n, ldq, ROLE_X));
  char* W = static_cast<char*>(h->Wws);
  const int64_t ldw = pad_ld(n_r);
  {
    GemmReq g{};
    g.conj = false; g.tA = &tV; g.tX = &tY; g.a3d = a3dV;
    g.M = (int)n_r; g.N = n; g.K = n;
    g.out = W; g.ldo = ldw; g.alpha = 1.0;
    ProfScope ps(h, CAT_TRSM, 1);
    STATUS_TRY(run_gemm(h, g));
  }
  CUDA_TRY(cudaMemcpy2DAsync(V, ldv * es, W, ldw * es, n_r * es, n, cudaMemcpyDeviceToDevice, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (sweeps_out) *sweeps_out = sweeps;
  if (!converged)
    fprintf(stderr, "[chase] rayleigh_ritz: Jacobi not converged after %d sweeps (off %.3e, ||A|| %.3e)\n",
            sweeps, std::sqrt(off[0]), std::sqrt(off[1]));
  return converged ? CHASE_OK : CHASE_ENOCONV;
}

double chase_shift_value(int64_t m, int64_t n, double norm) {
  return 11.0 * (double)(m * n + n * (n + 1)) * 1.1102230246251565e-16 * norm;
}

double chase_cond_est(const double* ritz, int64_t n, double c, double e, const int32_t* degrees,
                      int64_t locked) {
  if (!ritz || !degrees || n < 1 || locked < 0 || locked >= n || !(e > 0.0)) return NAN;
  const double tp = (ritz[0] - c) / e;
  const double t = (ritz[locked] - c) / e;
  // |rho| = max |t -+ sqrt(t^2 - 1)|: for |t| <= 1 both roots have modulus 1
  auto rho = [](double x) { return std::fabs(x) <= 1.0 ? 1.0 : std::fabs(x) + std::sqrt(x * x - 1.0); };
  const int32_t d = degrees[locked];
  int32_t dM = d;
  for (int64_t j = locked; j < n; ++j) dM = std::max(dM, degrees[j]);
  return std::pow(rho(t), (double)d) * std::pow(rho(tp), (double)(dM - d));
}

chase_status_t chase_profile_enable(chase_handle_t h, int enable) {
  if (!h) return CHASE_EINVAL;
  h->profiling = enable != 0;
  return CHASE_OK;
}

chase_status_t chase_profile_read(chase_handle_t h, double ms[8], int64_t launches[8]) {
  if (!h || !ms || !launches) return CHASE_EINVAL;
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  for (int i = 0; i < 8; ++i) {
    ms[i] = 0.0;
    launches[i] = 0;
  }
  for (auto& ev : h->evs) {
    float t = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&t, ev.a, ev.b));
    ms[ev.cat] += t;
    h->pool.push_back(ev.a);
    h->pool.push_back(ev.b);
  }
  h->evs.clear();
  for (int i = 0; i < CAT_N; ++i) {
    launches[i] = h->launches[i];
    h->launches[i] = 0;
  }
  return CHASE_OK;
}

chase_status_t chase_destroy(chase_handle_t h) {
  if (!h) return CHASE_EINVAL;
  if (h->rcomm) ncclCommDestroy(h->rcomm);
  if (h->ccomm) ncclCommDestroy(h->ccomm);
  if (h->world) ncclCommDestroy(h->world);
  for (auto& ev : h->evs) {
    cudaEventDestroy(ev.a);
    cudaEventDestroy(ev.b);
  }
  for (auto e : h->pool) cudaEventDestroy(e);
  if (h->h_info) cudaFreeHost(h->h_info);
  if (h->h_shift) cudaFreeHost(h->h_shift);
  delete h;
  return CHASE_OK;
}

}  // extern "C"

#include "solver.inc"
