// liblbm19 -- B200-native D3Q19 fused pull stream + BGK collide (sm_100a).
//
// Drop-in replacement for the reference's compiled step operator
// (pkg/src/sparselbm/kernel.py:56-141) and the Simulation plumbing around it;
// the C-ABI is declared in include/lbm19.h.  Kernels:
//
//   k_flags        node descriptors -> packed u32 flag word per slot (mask,
//                  type, orientation, bc index); layouts.py:173-188 on device
//   k_tile_keep / k_tile_compact
//                  sparse tile index: kept-tile flags, exclusive scan (CUB),
//                  compacted (tx,ty,tz) list and the 27-entry neighbour table
//                  (layouts.py:263-269, 389-401 generalised)
//   k_init         float64 equilibrium, cast to the storage type (kernel.py:190-237)
//   k_step_dense   ONE fused pass per step: pull gather with link-wise bounce-back,
//                  Zou-He closures, moments, BGK, node-local store (kernel.py:72-141)
//   k_step_tile    the same over the compacted tile list + nbr27
//   k_macro / k_mass / k_nonfinite / k_get_pdf / k_set_pdf   readbacks
//
// Storage (HBM): two buffers, each (19, plane_stride) in the storage type.
//   dense: slot(x,y,z) = ((z+1)*ny + y)*nxp + x, nxp = nx rounded up to 32,
//          one ghost plane below and above (z-slab halos / periodic wrap);
//   tile:  slot = rank*TN + ((lz*ey + ly)*ex + lx), each (tile, direction)
//          block contiguous (8^3 fp32 -> 2 KB).
#include <cuda_runtime.h>

#include <nvtx3/nvToolsExt.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <cstring>
#include <unistd.h>
#include <sys/mman.h>
#include <string>
#include <thread>
#include <vector>

#include "d3q19.cuh"
#include "lbm19.h"

using namespace lbm;

// NVTX ranges (header-only NVTX3; no-ops unless a tool such as nsys/ncu attaches)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// ------------------------------------------------------------ error plumbing
static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      if (e_ == cudaErrorMemoryAllocation) {                                          \
        cudaGetLastError();                                                           \
        return fail(LBM_ENOMEM, "%s: %s", #call, cudaGetErrorString(e_));             \
      }                                                                               \
      return fail(LBM_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                          \
    }                                                                                 \
  } while (0)

#define CKL() CK(cudaGetLastError())

#include "layout.cuh"
#include "geometry_kernels.cuh"
#include "readback_kernels.cuh"
#include "step_dense.cuh"
#include "step_tiles.cuh"

// ----------------------------------------------------------------- handle
struct lbm_handle {
  lbm_desc d{};
  int esize = 4;
  Geo g{};
  SlotMap sm{nullptr};
  long long n_nodes = 0, n_slots = 0, nflags = 0;
  long long n_tiles = 0, ntiles_grid = 0;
  long long n_nonsolid = 0;
  void* f[2] = {nullptr, nullptr};
  uint32_t* flags = nullptr;
  int* rank = nullptr;    // tile rank grid
  int* tiles = nullptr;   // (T, 3)
  int* nbr27 = nullptr;   // (T, 27)
  void* gh[2] = {nullptr, nullptr};  // tile slabs: ghost planes per buffer, [lo | hi] x 5 x ny x nx
  uint32_t* items = nullptr;  // warp work list, 4 words per warp (tile, brick bytes x2, uniform | count), MODE 5/8
  unsigned long long* lut = nullptr;  // per in-tile slot neighbour deltas (TileUpLUT)
  int n_items = 0;
  int n_items_b = 0;        // z-slabs: the first n_items_b items hold the boundary tile planes
  bool auto_wlist = false;  // default tile kernel = warp work list (sparse tiles)
  bool wlist_ok = false;    // work-list items fit their packing (<= 8 brick groups per warp)
  double live_frac = 1.0;   // live bricks / brick slots of the kept tiles
  bool has_glo = false, has_ghi = false;  // tile slabs: links cross z = -1 / z = nz
  uint32_t* bmask = nullptr;  // (T, 4) live-brick bit masks
  uint32_t* ubits = nullptr;  // dense: uniform-chunk bitmap (1 bit per 32 nodes)
  bool use_ubits = true;
  long long meta_bytes = 0;   // flag / index bytes one step reads
  void* bcv = nullptr;    // (nb, 3) storage type
  void* bcr = nullptr;    // (nb) storage type
  uint8_t* bckind64 = nullptr;
  double* bcv64 = nullptr;
  double* bcr64 = nullptr;
  int nb = 0;
  int parity = 0;
  int variant = 0;  // step-kernel variant (LBM_STEP_VARIANT), see launch_step
  bool variant_set = false;  // LBM_STEP_VARIANT given: no automatic choice
  bool geometry = false, initialized = false;
  long long step_count = 0, visited_total = 0, launches = 0;
  long long device_bytes = 0;
  double last_ms = 0.0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  void* pin[2] = {nullptr, nullptr};   // pinned host staging for pipelined readbacks
  size_t pin_bytes = 0;
  cudaEvent_t evc[2] = {nullptr, nullptr};
  double* scratch = nullptr;   // reductions
  unsigned long long* uscratch = nullptr;
  // z-slab halo (fused peer stores); see k_step_dense and lbm_halo_connect
  struct Peer {
    bool on = false, ipc = false;
    void* f[2] = {nullptr, nullptr};
    int* rank = nullptr;   // tile A-A slabs: the neighbour's tile rank grid (peer memory)
    unsigned long long* sync = nullptr;
    long long ps = 0;
    int nz = 0;
  } lo, hi;
  unsigned long long* sync = nullptr;  // [0] written by the lower, [1] by the upper neighbour
  int* herr = nullptr;
  bool halo_dirty = true;
  bool pending = false;                // lbm_step_async issued, not yet synchronised
  cudaGraphExec_t graph[2] = {nullptr, nullptr};  // kGraphSteps steps from parity 0 / 1
  long long graph_launches = 0;                    // kernel launches per graph replay
  bool use_graph = true;
};

constexpr int kGraphSteps = 32;

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int ilog2(int v) {
  int l = 0;
  while ((1 << l) < v) ++l;
  return l;
}

template <typename P>
int dev_alloc(lbm_handle* h, P** p, size_t bytes) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, bytes ? bytes : 16);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? LBM_ENOMEM : LBM_ECUDA,
                "cudaMalloc(%zu bytes): %s", bytes, cudaGetErrorString(e));
  }
  h->device_bytes += (long long)bytes;
  *p = (P*)q;
  return 0;
}

void dev_free(void* p) {
  if (p) cudaFree(p);
}

// Setup temporaries and readback staging come from the stream-ordered pool
// (cudaMallocAsync / cudaFreeAsync on the solver stream): no device-wide
// synchronisation per free, and the pool keeps the memory for the next
// handle -- after a large cudaFree, plain cudaMalloc / cudaFree of these
// buffers measured 20-600 ms (profiles/setup_phases_r02*.txt).
template <typename P>
int tmp_alloc(lbm_handle* h, P** p, size_t bytes) {
  void* q = nullptr;
  cudaError_t e = cudaMallocAsync(&q, bytes ? bytes : 16, h->stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? LBM_ENOMEM : LBM_ECUDA, "cudaMallocAsync(%zu bytes): %s", bytes,
                cudaGetErrorString(e));
  }
  *p = (P*)q;
  return 0;
}

void tmp_free(const lbm_handle* h, void* p) {
  if (p) cudaFreeAsync(p, h->stream);
}

// keep freed pool memory cached for the next temporaries (once per device)
void keep_pool(int device) {
  static bool done[64] = {};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    unsigned long long keep = 4ull << 30;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  done[device] = true;
}

// Copies of state the solver stream touches go through that stream: the
// legacy default stream does not order against a non-blocking stream, and a
// pageable cudaMemcpy can return before its DMA has landed.
cudaError_t scopy(const lbm_handle* h, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  return e;
}

void drop_graphs(lbm_handle* h) {
  for (int p = 0; p < 2; ++p)
    if (h->graph[p]) {
      cudaGraphExecDestroy(h->graph[p]);
      h->graph[p] = nullptr;
    }
}

void free_geometry(lbm_handle* h) {
  drop_graphs(h);
  dev_free(h->f[0]);
  dev_free(h->f[1]);
  dev_free(h->flags);
  dev_free(h->rank);
  dev_free(h->tiles);
  dev_free(h->nbr27);
  dev_free(h->items);
  h->items = nullptr;
  dev_free(h->lut);
  h->lut = nullptr;
  h->n_items = 0;
  h->n_items_b = 0;
  h->wlist_ok = h->auto_wlist = false;
  dev_free(h->gh[0]);
  dev_free(h->gh[1]);
  h->gh[0] = h->gh[1] = nullptr;
  dev_free(h->bmask);
  dev_free(h->ubits);
  dev_free(h->bcv);
  dev_free(h->bcr);
  dev_free(h->bckind64);
  dev_free(h->bcv64);
  dev_free(h->bcr64);
  h->f[0] = h->f[1] = nullptr;
  h->flags = nullptr;
  h->rank = h->tiles = h->nbr27 = nullptr;
  h->bmask = nullptr;
  h->ubits = nullptr;
  h->bcv = h->bcr = nullptr;
  h->bckind64 = nullptr;
  h->bcv64 = h->bcr64 = nullptr;
  h->device_bytes = 0;
  h->geometry = h->initialized = false;
}

bool is_tiled(int layout) { return layout == LBM_LAYOUT_TILE || layout == LBM_LAYOUT_POINTER_TILE; }

// elements of one PDF buffer: 19 planes of ps (tiles: T tiles x 19 blocks),
// plus, on tile A-A z-slabs, the 2 x 5 mirror planes of the cross-cut pushes
long long buf_elems(const lbm_handle* h) {
  const bool mirror = h->g.tiled && h->g.aa && (h->has_glo || h->has_ghi);
  return (long long)Q * h->g.ps + (mirror ? 10LL * h->g.nx * h->g.ny : 0LL);
}

dim3 node_grid(const Geo& g, int bx) { return dim3((g.nx + bx - 1) / bx, g.ny, g.nz); }

// peer ghost planes of buffer q (lockstep: every slab is at the same parity)
template <typename T>
Halo<T> make_halo(const lbm_handle* h, int q) {
  Halo<T> H{};
  if (h->g.aa) {
    // A-A: the neighbours' boundary planes themselves (lower slab's top plane,
    // upper slab's plane 0) -- the neighbour step reads and writes them directly
    for (int j = 0; j < 5; ++j) {
      H.lo[j] = h->lo.on ? (T*)h->lo.f[0] + (size_t)kZm(j) * h->lo.ps + (size_t)h->lo.nz * h->g.plane : nullptr;
      H.hi[j] = h->hi.on ? (T*)h->hi.f[0] + (size_t)kZp(j) * h->hi.ps + (size_t)h->g.plane : nullptr;
    }
    return H;
  }
  for (int j = 0; j < 5; ++j) {
    H.lo[j] = h->lo.on ? (T*)h->lo.f[q] + (size_t)kZm(j) * h->lo.ps + (size_t)(h->lo.nz + 1) * h->g.plane
                       : nullptr;
    H.hi[j] = h->hi.on ? (T*)h->hi.f[q] + (size_t)kZp(j) * h->hi.ps : nullptr;
  }
  return H;
}

template <typename T>
TileHalo<T> make_tile_halo(const lbm_handle* h, int q_pre, int q_post) {
  TileHalo<T> TH{};
  TH.on = h->g.tiled && h->gh[0] != nullptr;
  if (!TH.on) return TH;
  const size_t pn = (size_t)h->g.nx * h->g.ny;
  TH.tiles = h->tiles;
  TH.pre_lo = h->has_glo ? (const T*)h->gh[q_pre] : nullptr;
  TH.pre_hi = h->has_ghi ? (const T*)h->gh[q_pre] + 5 * pn : nullptr;
  for (int j = 0; j < 5; ++j) {
    TH.push_lo[j] = h->lo.on ? (T*)h->lo.f[q_post] + (5 + j) * pn : nullptr;
    TH.push_hi[j] = h->hi.on ? (T*)h->hi.f[q_post] + j * pn : nullptr;
  }
  return TH;
}

bool halo_on(const lbm_handle* h) { return h->lo.on || h->hi.on; }

// buffer holding the reference's `pre` (AA: the single in-place buffer)
void* pre_buf(const lbm_handle* h) { return h->g.aa ? h->f[0] : h->f[h->parity]; }

// Geo for readback launches: carries the AA state phase
Geo rb_geo(const lbm_handle* h) {
  Geo g = h->g;
  g.aph = h->g.aa ? h->parity : 0;
  return g;
}

long long visits_per_step(const lbm_handle* h) {
  return (h->d.layout == LBM_LAYOUT_DENSE) ? h->n_nodes
         : (h->d.layout == LBM_LAYOUT_BITMASK_NODE) ? h->n_nonsolid
                                                     : h->n_slots;
}

void halo_signal(lbm_handle* h) {
  h->launches += 1;
  k_halo_signal<<<1, 1, 0, h->stream>>>(h->lo.on ? h->lo.sync + 1 : nullptr,
                                         h->hi.on ? h->hi.sync + 0 : nullptr, h->sync + 2);
}

void halo_wait(lbm_handle* h) {
  h->launches += 1;
  k_halo_wait<<<1, 1, 0, h->stream>>>(h->sync, h->lo.on, h->hi.on, h->herr);
}


template <typename T>
void halo_push(lbm_handle* h) {
  if (h->g.tiled) {
    const TileHalo<T> TH = make_tile_halo<T>(h, h->parity, h->parity);
    h->launches += 1;
    k_tile_halo_push<T><<<dim3((h->g.nx + 127) / 128, h->g.ny), 128, 0, h->stream>>>((const T*)h->f[h->parity], h->sm,
                                                                                     h->g, TH);
    return;
  }
  const Halo<T> H = make_halo<T>(h, h->parity);
  h->launches += 1;
  dim3 grid((h->g.nxp + 127) / 128, h->g.ny);
  k_halo_push<T><<<grid, 128, 0, h->stream>>>((const T*)h->f[h->parity], H, h->g);
}

// TMA-staged tile kernel (variant 9): AB, whole-domain handles
bool tma_ok(const lbm_handle* h) { return h->g.tiled && !h->g.aa && h->gh[0] == nullptr; }

template <typename T, int TN>
void launch_tiles_tma(lbm_handle* h, const T* pre, T* post) {
  using C = TmaCfg<T, TN>;
  static int blocks = 0;  // resident CTAs per SM (per instantiation; same device family)
  static int sms = 0;
  if (!blocks) {
    cudaFuncSetAttribute(k_step_tiles_tma<T, TN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_step_tiles_tma<T, TN>, C::THREADS, C::SMEM);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->d.device);
    if (blocks < 1) blocks = 1;
  }
  long long grid = (long long)blocks * sms;
  if (grid > h->n_tiles) grid = h->n_tiles;
  k_step_tiles_tma<T, TN><<<(unsigned)grid, C::THREADS, C::SMEM, h->stream>>>(
      pre, post, h->flags, h->nbr27, (const T*)h->bcv, (const T*)h->bcr, h->g, (T)h->d.omega, h->bmask,
      (const ulonglong2*)h->lut, (int)h->n_tiles);
}

// part (z-slabs on the work list): 0 every item, 1 the boundary tile planes
// (with the ghost exchange), 2 the interior items
template <typename T, int TN>
void launch_tiles(lbm_handle* h, const T* pre, T* post, int part = 0) {
  constexpr int BT = TN < 256 ? TN : 256;
  const TileHalo<T> TH = make_tile_halo<T>(h, h->parity, 1 - h->parity);
  constexpr int M = sizeof(T) == 4 ? (1536 / BT > 32 ? 32 : 1536 / BT) : (768 / BT);
  constexpr int MS = M * 5 / 6 > 0 ? M * 5 / 6 : 1;  // select / ghost variants need more registers
  constexpr int MW = sizeof(T) == 4 ? 6 : 3;          // work list: 48 (fp32) resident warps per SM
  const unsigned nt = (unsigned)h->n_tiles;
  const T* bv = (const T*)h->bcv;
  const T* br = (const T*)h->bcr;
  const T om = (T)h->d.omega;
  const ulonglong2* lut = (const ulonglong2*)h->lut;
  // kernel choice by live-brick fraction (measured, profiles/sparse_r01.md):
  // < 0.85 the warp work list with exact per-link select; fuller tiles one
  // CTA per tile with speculative gathers + bounce-back fix-up.  z-slabs run
  // the same kernels with the ghost-plane exchange compiled in.
  const bool wl = h->wlist_ok && (h->variant_set ? h->variant == 8 : h->auto_wlist);
  if (h->variant_set && h->variant == 9 && tma_ok(h)) {
    launch_tiles_tma<T, TN>(h, pre, post);
    return;
  }
  if (wl) {
    if (!h->n_items) return;
    const uint4* it = (const uint4*)h->items;
    if (TH.on && part != 0) {
      const int i0 = part == 1 ? 0 : h->n_items_b, n = part == 1 ? h->n_items_b : h->n_items - h->n_items_b;
      if (n <= 0) return;
      const unsigned nbk = (unsigned)((n + kWarpsPerBlock - 1) / kWarpsPerBlock);
      if (part == 1)  // the ghost exchange needs 48 registers (fp32)
        k_step_tiles_w<T, TN, MW * 5 / 6, true><<<nbk, 32 * kWarpsPerBlock, 0, h->stream>>>(
            pre, post, h->flags, h->nbr27, bv, br, h->g, om, it + i0, n, lut, TH);
      else
        k_step_tiles_w<T, TN, MW><<<nbk, 32 * kWarpsPerBlock, 0, h->stream>>>(pre, post, h->flags, h->nbr27, bv, br,
                                                                              h->g, om, it + i0, n, lut);
      return;
    }
    const unsigned nb = (unsigned)((h->n_items + kWarpsPerBlock - 1) / kWarpsPerBlock);
    if (TH.on)  // the ghost exchange needs 48 registers (fp32)
      k_step_tiles_w<T, TN, MW * 5 / 6, true><<<nb, 32 * kWarpsPerBlock, 0, h->stream>>>(
          pre, post, h->flags, h->nbr27, bv, br, h->g, om, it, h->n_items, lut, TH);
    else
      k_step_tiles_w<T, TN, MW><<<nb, 32 * kWarpsPerBlock, 0, h->stream>>>(pre, post, h->flags, h->nbr27, bv, br,
                                                                           h->g, om, it, h->n_items, lut);
    return;
  }
  if (TH.on)
    k_step_tiles_x<T, TN, MS, true, true><<<nt, BT, 0, h->stream>>>(pre, post, h->flags, h->nbr27, bv, br, h->g, om,
                                                                     h->bmask, lut, TH);
  else
    k_step_tiles_x<T, TN, M><<<nt, BT, 0, h->stream>>>(pre, post, h->flags, h->nbr27, bv, br, h->g, om, h->bmask, lut);
}

template <typename T>
TileAAHalo<T> make_tile_aa_halo(const lbm_handle* h) {
  TileAAHalo<T> AH{};
  const Geo& g = h->g;
  const long long row = (long long)g.gy * g.gx;
  if (h->lo.on) {
    AH.f_lo = (T*)h->lo.f[0];
    AH.rank_lo = h->lo.rank + (long long)((h->lo.nz - 1) >> g.lez) * row;
    AH.lz_lo = (h->lo.nz - 1) & (g.ez - 1);
  }
  if (h->hi.on) {
    AH.f_hi = (T*)h->hi.f[0];
    AH.rank_hi = h->hi.rank;  // its tile plane 0
  }
  AH.mirror = (T*)h->f[0] + (size_t)Q * g.ps;
  AH.tiles = h->tiles;
  return AH;
}

template <typename T, int TN>
void launch_tiles_aa(lbm_handle* h, T* F) {
  constexpr int BT = TN < 256 ? TN : 256;
  constexpr int M = sizeof(T) == 4 ? (1536 / BT > 32 ? 32 : 1536 / BT) : (768 / BT);
  const unsigned nt = (unsigned)h->n_tiles;
  const T* bv = (const T*)h->bcv;
  const T* br = (const T*)h->bcr;
  const T om = (T)h->d.omega;
  const ulonglong2* lut = (const ulonglong2*)h->lut;
  constexpr int MN = M * 5 / 6 > 0 ? M * 5 / 6 : 1;  // neighbour step: looser register cap (48)
  // the warp work list where the AB step would use it
  const bool wl = h->wlist_ok && (h->variant_set ? h->variant == 8 : h->auto_wlist);
  if (wl) {
    if (!h->n_items) return;
    const unsigned nb = (unsigned)((h->n_items + kWarpsPerBlock - 1) / kWarpsPerBlock);
    const uint4* it = (const uint4*)h->items;
    // 48 resident warps for both phases (40 registers; the neighbour step
    // spills 8 B and still measured 0-1 % faster than 40 warps at 48
    // registers, profiles/ab_aa_warp_list_r01.txt)
    if (h->parity == 0 && halo_on(h)) {
      // z-slab: the boundary tile planes' items (ordered first) reach into the
      // neighbours; the interior items run the plain neighbour step
      const int nbi = h->n_items_b, nin = h->n_items - h->n_items_b;
      if (nbi > 0)
        k_step_tiles_aa_w<T, TN, 1, sizeof(T) == 4 ? 5 : 2, true>
            <<<(unsigned)((nbi + kWarpsPerBlock - 1) / kWarpsPerBlock), 32 * kWarpsPerBlock, 0, h->stream>>>(
                F, h->flags, h->nbr27, bv, br, h->g, om, it, nbi, lut, make_tile_aa_halo<T>(h));
      if (nin > 0)
        k_step_tiles_aa_w<T, TN, 1, sizeof(T) == 4 ? 6 : 3>
            <<<(unsigned)((nin + kWarpsPerBlock - 1) / kWarpsPerBlock), 32 * kWarpsPerBlock, 0, h->stream>>>(
                F, h->flags, h->nbr27, bv, br, h->g, om, it + nbi, nin, lut);
    } else if (h->parity == 0)
      k_step_tiles_aa_w<T, TN, 1, sizeof(T) == 4 ? 6 : 3><<<nb, 32 * kWarpsPerBlock, 0, h->stream>>>(
          F, h->flags, h->nbr27, bv, br, h->g, om, it, h->n_items, lut);
    else
      k_step_tiles_aa_w<T, TN, 0, sizeof(T) == 4 ? 6 : 3><<<nb, 32 * kWarpsPerBlock, 0, h->stream>>>(
          F, h->flags, h->nbr27, bv, br, h->g, om, it, h->n_items, lut);
    return;
  }
  if (h->parity == 0 && halo_on(h))
    k_step_tiles_aa<T, TN, 1, (MN * 5 / 6 > 0 ? MN * 5 / 6 : 1), true><<<nt, BT, 0, h->stream>>>(
        F, h->flags, h->nbr27, bv, br, h->g, om, h->bmask, lut, make_tile_aa_halo<T>(h));
  else if (h->parity == 0)
    k_step_tiles_aa<T, TN, 1, MN><<<nt, BT, 0, h->stream>>>(F, h->flags, h->nbr27, bv, br, h->g, om, h->bmask, lut);
  else
    k_step_tiles_aa<T, TN, 0, M><<<nt, BT, 0, h->stream>>>(F, h->flags, h->nbr27, bv, br, h->g, om, h->bmask, lut);
}

// grid z-extent of a dense launch covering `zmode`'s planes (slab_z)
unsigned zmode_planes(const Geo& g, int zmode) {
  return zmode == 0 ? (unsigned)g.nz : (zmode == 1 ? (g.nz > 1 ? 2u : 1u) : (g.nz > 2 ? (unsigned)g.nz - 2u : 0u));
}

// one step from `pre` into `post` (AB); AA updates `post` (== pre) in place.
// zmode (dense z-slabs): 0 every plane, 1 the two boundary planes, 2 the interior
template <typename T>
int launch_step(lbm_handle* h, const void* pre, void* post, int zmode = 0) {
  const Geo& g = h->g;
  const T om = (T)h->d.omega;
  Planes<T> P;
  for (int i = 0; i < Q; ++i) {
    P.pre[i] = (const T*)pre + (size_t)i * g.ps;
    P.post[i] = (T*)post + (size_t)i * g.ps;
  }
  constexpr int D1 = sizeof(T) == 4 ? 12 : 6;
#ifdef LBM_EXPERIMENTS
  // variants (LBM_STEP_VARIANT): 1 warp-uniform fast path else per-link
  // select; 2 / 3 the same with a looser register cap; 8 the 128-bit kernel
  const int var = h->variant;
  constexpr int D2 = sizeof(T) == 4 ? 10 : 5;
  constexpr int V4B = 3;  // 128-bit kernel: 3 x 128 threads per SM, up to 168 registers
#endif
  const T* bv = (const T*)h->bcv;
  const T* br = (const T*)h->bcr;
  if (g.aa) {
    // parity = AA state phase: 0 -> neighbour step, 1 -> node-local step
    if (!g.tiled) {
      Planes1<T> F;
      for (int i = 0; i < Q; ++i) F.f[i] = (T*)post + (size_t)i * g.ps;
      dim3 grid((g.nxp + 127) / 128, g.ny, zmode_planes(g, zmode));
      if (grid.z == 0) return 0;
      Halo<T> H = h->parity == 0 ? make_halo<T>(h, 0) : Halo<T>{};
      H.zmode = zmode;
      if (h->parity == 0) {
#ifdef LBM_EXPERIMENTS
        if (h->variant == 12)  // row-aligned pushes through shared memory (measured slower)
          k_step_dense_aa_nb<T, D1><<<grid, 128, 0, h->stream>>>(F, h->flags, h->ubits, bv, br, g, om, H);
        else
#endif
        k_step_dense_aa<T, 1, D1><<<grid, 128, 0, h->stream>>>(F, h->flags, h->ubits, bv, br, g, om, H);
      } else
        k_step_dense_aa<T, 0, D1><<<grid, 128, 0, h->stream>>>(F, h->flags, h->ubits, bv, br, g, om, H);
    } else {
      if (h->n_tiles == 0) return 0;
      switch (g.tn) {
        case 32: launch_tiles_aa<T, 32>(h, (T*)post); break;
        case 64: launch_tiles_aa<T, 64>(h, (T*)post); break;
        case 128: launch_tiles_aa<T, 128>(h, (T*)post); break;
        case 256: launch_tiles_aa<T, 256>(h, (T*)post); break;
        default: launch_tiles_aa<T, 512>(h, (T*)post); break;
      }
    }
    h->launches += 1;
    return 0;
  }
  if (!g.tiled) {
    const int bx = 128;
    dim3 grid((g.nxp + bx - 1) / bx, g.ny, zmode_planes(g, zmode));
    if (grid.z == 0) return 0;
    Halo<T> H = make_halo<T>(h, 1 - h->parity);
    H.zmode = zmode;
#ifdef LBM_EXPERIMENTS
    // measured-slower alternatives, built only into the experiments library
    // (python -m paper_2108_13241_b200.build --experiments; profiles/v4_r01.md)
    if (var == 1)
      k_step_dense<T, 1, D1><<<grid, bx, 0, h->stream>>>(P, h->flags, h->ubits, bv, br, g, om, H);
    else if (var == 2)
      k_step_dense<T, 0, D2><<<grid, bx, 0, h->stream>>>(P, h->flags, h->ubits, bv, br, g, om, H);
    else if (var == 3)
      k_step_dense<T, 1, D2><<<grid, bx, 0, h->stream>>>(P, h->flags, h->ubits, bv, br, g, om, H);
    else if (var == 8 && sizeof(T) == 4 && !halo_on(h)) {
      Planes<float> P4;
      for (int i = 0; i < Q; ++i) {
        P4.pre[i] = (const float*)P.pre[i];
        P4.post[i] = (float*)P.post[i];
      }
      const dim3 g4((g.nxp / 4 + 127) / 128, g.ny, g.nz);
      k_step_dense_v4<V4B><<<g4, 128, 0, h->stream>>>(P4, h->flags, h->ubits, (const float*)bv, (const float*)br, g,
                                                       (float)om);
    }
    else
#endif
      k_step_dense<T, 0, D1><<<grid, bx, 0, h->stream>>>(P, h->flags, h->ubits, bv, br, g, om, H);
  } else {
    if (h->n_tiles == 0) return 0;
    switch (g.tn) {
      case 32: launch_tiles<T, 32>(h, (const T*)pre, (T*)post, zmode); break;
      case 64: launch_tiles<T, 64>(h, (const T*)pre, (T*)post, zmode); break;
      case 128: launch_tiles<T, 128>(h, (const T*)pre, (T*)post, zmode); break;
      case 256: launch_tiles<T, 256>(h, (const T*)pre, (T*)post, zmode); break;
      default: launch_tiles<T, 512>(h, (const T*)pre, (T*)post, zmode); break;
    }
  }
  h->launches += 1;
  return 0;
}

// one step of a connected z-slab: wait for the neighbours' previous step,
// then the boundary planes (dense) / boundary tile planes (work list), the
// signal, and the interior -- the neighbours' next step overlaps this slab's
// interior.  Safe because only boundary-plane threads touch the ghost planes
// (AB) or the neighbour's boundary plane (A-A), and the signal follows them.
template <typename T>
void slab_step(lbm_handle* h, const void* pre, void* post) {
  halo_wait(h);
  // dense (AB and A-A) always; tile slabs when they run the work list (its
  // items are ordered boundary tile planes first)
  const bool split = !h->g.tiled || (!h->g.aa && h->wlist_ok && (h->variant_set ? h->variant == 8 : h->auto_wlist));
  if (split) {
    launch_step<T>(h, pre, post, 1);
    halo_signal(h);
    launch_step<T>(h, pre, post, 2);
  } else {
    launch_step<T>(h, pre, post);
    halo_signal(h);
  }
}

// CUDA lazy module loading loads a kernel at its first launch, and loading
// waits for the device: with a neighbour's k_halo_wait spinning, that first
// launch would stall until the wait times out.  A slab therefore loads every
// kernel its step loop can launch when it is connected, before any spins.
template <typename T, int TN>
void preload_tiles(cudaFuncAttributes* a) {
  constexpr int BT = TN < 256 ? TN : 256;
  constexpr int M = sizeof(T) == 4 ? (1536 / BT > 32 ? 32 : 1536 / BT) : (768 / BT);
  constexpr int MN = M * 5 / 6 > 0 ? M * 5 / 6 : 1;
  cudaFuncGetAttributes(a, k_step_tiles_aa<T, TN, 1, (MN * 5 / 6 > 0 ? MN * 5 / 6 : 1), true>);
  cudaFuncGetAttributes(a, k_step_tiles_aa<T, TN, 0, M>);
  cudaFuncGetAttributes(a, k_step_tiles_aa_w<T, TN, 1, sizeof(T) == 4 ? 5 : 2, true>);
  cudaFuncGetAttributes(a, k_step_tiles_aa_w<T, TN, 0, sizeof(T) == 4 ? 6 : 3>);
  cudaFuncGetAttributes(a, k_step_tiles_w<T, TN, sizeof(T) == 4 ? 6 : 3>);
  cudaFuncGetAttributes(a, k_step_tiles_x<T, TN, (M * 5 / 6 > 0 ? M * 5 / 6 : 1), true, true>);
  cudaFuncGetAttributes(a, k_step_tiles_w<T, TN, (sizeof(T) == 4 ? 6 : 3) * 5 / 6, true>);
}

template <typename T>
void preload_halo_kernels(const lbm_handle* h) {
  constexpr int D1 = sizeof(T) == 4 ? 12 : 6;
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_halo_wait);
  cudaFuncGetAttributes(&a, k_halo_signal);
  if (!h->g.tiled && h->g.aa) {
    cudaFuncGetAttributes(&a, k_step_dense_aa<T, 1, D1>);
    cudaFuncGetAttributes(&a, k_step_dense_aa<T, 0, D1>);
  } else if (!h->g.tiled) {
    cudaFuncGetAttributes(&a, k_halo_push<T>);
    cudaFuncGetAttributes(&a, k_step_dense<T, 0, D1>);
  } else {
    cudaFuncGetAttributes(&a, k_tile_halo_push<T>);
    switch (h->g.tn) {
      case 32: preload_tiles<T, 32>(&a); break;
      case 64: preload_tiles<T, 64>(&a); break;
      case 128: preload_tiles<T, 128>(&a); break;
      case 256: preload_tiles<T, 256>(&a); break;
      default: preload_tiles<T, 512>(&a); break;
    }
  }
  cudaGetLastError();
}

}  // namespace

// -------------------------------------------- pipelined host <-> device copies
// Pinned staging slots are kept in a small process-wide cache when a handle
// is destroyed, so the next handle's first upload / readback does not pay
// cudaHostAlloc (pinning 2 x 64 MB costs tens of ms) -- like the CUDA
// context, the staging outlives one Simulation.
static std::mutex g_pin_mu;
static std::vector<std::pair<void*, size_t>> g_pin_cache;

static void release_pinned(void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  if (g_pin_cache.size() < 4) {
    g_pin_cache.emplace_back(p, bytes);
    return;
  }
  cudaFreeHost(p);
}

// both staging slots of h hold at least `bytes`
static int ensure_pinned(lbm_handle* h, size_t bytes) {
  if (h->pin_bytes >= bytes && h->pin[0] && h->pin[1]) return 0;
  for (int b = 0; b < 2; ++b) {
    release_pinned(h->pin[b], h->pin_bytes);
    h->pin[b] = nullptr;
  }
  h->pin_bytes = bytes;
  for (int b = 0; b < 2; ++b) {
    {
      std::lock_guard<std::mutex> lk(g_pin_mu);
      for (size_t k = 0; k < g_pin_cache.size(); ++k)
        if (g_pin_cache[k].second == bytes) {
          h->pin[b] = g_pin_cache[k].first;
          g_pin_cache.erase(g_pin_cache.begin() + (long)k);
          break;
        }
    }
    if (!h->pin[b] && cudaHostAlloc(&h->pin[b], bytes, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      h->pin[b] = nullptr;
      for (int q = 0; q < 2; ++q) {  // keep the slot that was obtained
        release_pinned(h->pin[q], bytes);
        h->pin[q] = nullptr;
      }
      h->pin_bytes = 0;
      return fail(LBM_ENOMEM, "pinned staging of %zu bytes failed", bytes);
    }
  }
  return 0;
}
// host copy split over threads (also spreads the page faults of fresh
// destination arrays)
__attribute__((visibility("hidden"))) void lbm_bulk_copy(char* d, const char* s, size_t n);  // host_copy.cpp

// Persistent copy workers, parked on a condition variable between calls: a
// readback copies 64 staging chunks, and spawning + joining 15 threads per
// chunk was a visible part of its host time.  Created on first use and never
// torn down (detached); one call at a time.
class CopyPool {
 public:
  explicit CopyPool(int workers) : nw_(workers) {
    for (int t = 1; t <= nw_; ++t) std::thread([this, t] { loop(t); }).detach();
  }
  int size() const { return nw_ + 1; }
  // runs f(0) .. f(nw) -- f(0) on the calling thread -- and returns when all finished
  void run(const std::function<void(int)>& f) {
    std::lock_guard<std::mutex> one(run_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &f;
      pending_ = nw_;
      ++gen_;
    }
    go_.notify_all();
    f(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  void loop(int t) {
    long seen = 0;
    for (;;) {
      const std::function<void(int)>* f;
      {
        std::unique_lock<std::mutex> lk(mu_);
        go_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        f = job_;
      }
      (*f)(t);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  const int nw_;
  std::mutex run_mu_, mu_;
  std::condition_variable go_, done_;
  const std::function<void(int)>* job_ = nullptr;
  long gen_ = 0;
  int pending_ = 0;
};

static void par_copy(const std::vector<std::pair<char*, const char*>>& dst_src, const std::vector<size_t>& n) {
  size_t total = 0;
  for (size_t v : n) total += v;
  static const int hw = [] {
    const unsigned c = std::thread::hardware_concurrency();
    return c == 0 ? 8 : (c > 16 ? 16 : (int)c);
  }();
  static const bool pooled = [] {
    const char* v = getenv("LBM_COPY_POOL");
    return !(v && v[0] == '0');
  }();
  const int nt = total > (8u << 20) ? hw : 1;
  const std::function<void(int)> work = [&](int t) {
    for (size_t k = 0; k < n.size(); ++k) {
      const size_t per = (n[k] + nt - 1) / nt, a = per * t, b = a + per < n[k] ? a + per : n[k];
      if (a < b) lbm_bulk_copy(dst_src[k].first + a, dst_src[k].second + a, b - a);
    }
  };
  if (nt == 1) {
    work(0);
    return;
  }
  if (pooled) {
    // leaked on purpose (detached workers outlive main); a forked child has no
    // workers, so it starts its own pool
    static std::mutex mu;
    static CopyPool* pool = nullptr;
    static pid_t owner = 0;
    CopyPool* p;
    {
      std::lock_guard<std::mutex> lk(mu);
      if (!pool || owner != getpid()) {
        pool = new CopyPool(hw - 1);
        owner = getpid();
      }
      p = pool;
    }
    p->run(work);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
}

// Fresh caller arrays (np.empty) fault their pages in on the first write, 4 KB
// at a time; asking for transparent huge pages first turns the readback's
// fault-in into 2 MB faults (no-op where THP is off).
static void advise_huge(void* p, size_t bytes) {
  static const bool off = [] {
    const char* v = getenv("LBM_THP");
    return v && v[0] == '0';
  }();
  if (off) return;
  const uintptr_t a = ((uintptr_t)p + (2u << 20) - 1) & ~(uintptr_t)((2u << 20) - 1);
  const uintptr_t e = ((uintptr_t)p + bytes) & ~(uintptr_t)((2u << 20) - 1);
  if (e > a) madvise((void*)a, e - a, MADV_HUGEPAGE);
}

// Pipelined device -> host readback in z chunks: chunk k's kernel and D2H
// copy (into pinned staging) overlap the host copy of chunk k-1 out of the
// other pinned slot.  launch(k, z0, nzc, dev) enqueues the chunk kernel;
// consume(k, z0, nzc, pinned) copies it into the caller's arrays.
template <class Launch, class Consume>
static int pipelined_d2h(lbm_handle* h, long long bytes_per_node, Launch launch, Consume consume) {
  const long long pn = (long long)h->g.nx * h->g.ny;
  const size_t want = 64u << 20;  // per staging slot
  long long cz = (long long)want / (pn * bytes_per_node);
  if (cz < 1) cz = 1;
  if (cz > h->g.nz) cz = h->g.nz;
  if (cz > 65535) cz = 65535;
  const size_t slot = (size_t)(cz * pn * bytes_per_node);
  const auto s0 = std::chrono::steady_clock::now();
  if (int rc_ = ensure_pinned(h, slot)) return rc_;
  for (int b = 0; b < 2; ++b)
    if (!h->evc[b]) CK(cudaEventCreateWithFlags(&h->evc[b], cudaEventDisableTiming));
  keep_pool(h->d.device);
  char* dev = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&dev, 2 * slot, h->stream);
  const auto s1 = std::chrono::steady_clock::now();
  if (e != cudaSuccess) return fail(LBM_ENOMEM, "readback staging: %s", cudaGetErrorString(e));
  const int nz = h->g.nz;
  const int nchunk = (int)((nz + cz - 1) / cz);
  const char* tv = getenv("LBM_TIMING");
  const bool timing = tv && tv[0] == '1';
  double t_wait = 0.0, t_cons = 0.0;
  for (int k = 0; k <= nchunk && e == cudaSuccess; ++k) {
    if (k < nchunk) {
      const int b = k & 1, z0 = (int)(k * cz), nzc = (int)(nz - z0 < cz ? nz - z0 : cz);
      launch(k, z0, nzc, dev + b * slot);
      e = cudaGetLastError();
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(h->pin[b], dev + b * slot, (size_t)(nzc * pn * bytes_per_node), cudaMemcpyDeviceToHost,
                            h->stream);
      if (e == cudaSuccess) e = cudaEventRecord(h->evc[b], h->stream);
    }
    if (k > 0 && e == cudaSuccess) {
      const int b = (k - 1) & 1, z0 = (int)((k - 1) * cz), nzc = (int)(nz - z0 < cz ? nz - z0 : cz);
      const auto w0 = std::chrono::steady_clock::now();
      e = cudaEventSynchronize(h->evc[b]);
      const auto w1 = std::chrono::steady_clock::now();
      if (e == cudaSuccess) consume(k - 1, z0, nzc, (const char*)h->pin[b]);
      t_wait += std::chrono::duration<double, std::milli>(w1 - w0).count();
      t_cons += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w1).count();
    }
  }
  const auto s2 = std::chrono::steady_clock::now();
  cudaFreeAsync(dev, h->stream);
  cudaStreamSynchronize(h->stream);
  if (timing) {
    const auto s3 = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    fprintf(stderr,
            "[lbm timing] readback: staging %.3f ms, %d chunks of %zu B (DMA wait %.3f ms, host copy %.3f ms), "
            "loop %.3f ms, teardown %.3f ms\n",
            ms(s0, s1), nchunk, slot, t_wait, t_cons, ms(s1, s2), ms(s2, s3));
  }
  if (e != cudaSuccess) return fail(LBM_ECUDA, "readback: %s", cudaGetErrorString(e));
  return 0;
}

// Pipelined host -> device upload through the pinned staging slots: the host
// copy of chunk k+1 (threads) overlaps the DMA of chunk k.
static int pipelined_h2d(lbm_handle* h, void* dev, const void* host, size_t bytes) {
  const size_t slot = 64u << 20;
  if (bytes < (4u << 20)) {  // small: one plain copy
    CK(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, h->stream));
    return 0;
  }
  if (int rc_ = ensure_pinned(h, slot)) return rc_;
  for (int b = 0; b < 2; ++b)
    if (!h->evc[b]) CK(cudaEventCreateWithFlags(&h->evc[b], cudaEventDisableTiming));
  const size_t n = (bytes + slot - 1) / slot;
  for (size_t k = 0; k < n; ++k) {
    const int b = (int)(k & 1);
    const size_t off = k * slot, len = bytes - off < slot ? bytes - off : slot;
    CK(cudaEventSynchronize(h->evc[b]));  // slot b's previous DMA (this or an earlier call) is done
    par_copy({{(char*)h->pin[b], (const char*)host + off}}, {len});
    CK(cudaMemcpyAsync((char*)dev + off, h->pin[b], len, cudaMemcpyHostToDevice, h->stream));
    CK(cudaEventRecord(h->evc[b], h->stream));
  }
  return 0;
}

// Descriptor upload packed on the host: type | orientation << 3 and the bc
// index byte (the flag word keeps 8 bits of it) -- 2 B per node on the wire
// instead of 6 -- range-checked while packing (threads), each chunk's DMA
// overlapping the packing of the next through the two pinned slots.
// err: bit 0 type / orientation out of range, bit 1 a velocity / pressure
// node without a valid bc index or orientation.
static int upload_descriptors(lbm_handle* h, uint8_t* dto, uint8_t* dbc, const uint8_t* type, const uint8_t* orient,
                              const int32_t* bc, long long N, int nb, int* err) {
  const size_t half = 32u << 20;  // nodes per chunk: 32 MB of each output per pinned slot
  if (int rc_ = ensure_pinned(h, 2 * half)) return rc_;
  for (int b = 0; b < 2; ++b)
    if (!h->evc[b]) CK(cudaEventCreateWithFlags(&h->evc[b], cudaEventDisableTiming));
  static const int hw = [] {
    const unsigned c = std::thread::hardware_concurrency();
    return c == 0 ? 8 : (c > 16 ? 16 : (int)c);
  }();
  std::vector<int> errs(hw, 0);
  const long long nchunk = (N + (long long)half - 1) / (long long)half;
  for (long long k = 0; k < nchunk; ++k) {
    const int b = (int)(k & 1);
    const long long off = k * (long long)half, n = N - off < (long long)half ? N - off : (long long)half;
    CK(cudaEventSynchronize(h->evc[b]));  // slot b's previous DMA is done
    uint8_t* pto = (uint8_t*)h->pin[b];
    uint8_t* pbc = pto + half;
    const int nt = n > (1 << 20) ? hw : 1;
    auto work = [&](int t) {
      const long long per = (n + nt - 1) / nt, a = per * t, e = a + per < n ? a + per : n;
      // branch-free so that the loop vectorises (host code is built with -O3)
      const uint8_t* __restrict__ ty_ = type + off;
      const uint8_t* __restrict__ or_ = orient + off;
      const int32_t* __restrict__ bc_ = bc + off;
      uint8_t* __restrict__ to_ = pto;
      uint8_t* __restrict__ bb_ = pbc;
      const uint32_t unb = (uint32_t)nb;
      uint32_t er = 0;
      for (long long i = a; i < e; ++i) {
        const uint32_t ty = ty_[i], o = or_[i];
        const int32_t bi = bc_[i];
        const uint32_t isbc = (ty - (uint32_t)VELOCITY_BC) <= 1u;  // VELOCITY_BC or PRESSURE_BC
        const uint32_t badb = (uint32_t)bi >= unb;                  // also bi < 0
        er |= (uint32_t)(ty > (uint32_t)PRESSURE_BC) | (uint32_t)(o > (uint32_t)O_BOTTOM) |
              ((isbc & (badb | (uint32_t)(o == (uint32_t)O_NONE))) << 1);
        to_[i] = (uint8_t)((ty & 7u) | ((o & 7u) << 3));
        bb_[i] = (uint8_t)(bi & ~(bi >> 31));                       // bc byte, negative -> 0
      }
      errs[t] |= (int)er;
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    CK(cudaMemcpyAsync(dto + off, pto, (size_t)n, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(dbc + off, pbc, (size_t)n, cudaMemcpyHostToDevice, h->stream));
    CK(cudaEventRecord(h->evc[b], h->stream));
  }
  for (int e : errs) *err |= e;
  return 0;
}

// ================================================================= C-ABI
extern "C" {

const char* lbm_last_error(void) { return g_err.c_str(); }
int lbm_abi_version(void) { return LBM_ABI_VERSION; }

int lbm_device_count(int* n) {
  if (!n) return fail(LBM_EINVAL, "n is NULL");
  CK(cudaGetDeviceCount(n));
  return 0;
}

int lbm_copy_bandwidth(int32_t device, int32_t layout, int64_t block_bytes, int32_t repetitions, int32_t warmup,
                       double* bytes_per_s) {
  if (!bytes_per_s) return fail(LBM_EINVAL, "bytes_per_s is NULL");
  if (block_bytes < 64 * 1024) return fail(LBM_EINVAL, "block_bytes must be at least 64 KiB, got %lld", (long long)block_bytes);
  if (repetitions < 1 || warmup < 0) return fail(LBM_EINVAL, "need repetitions >= 1 and warmup >= 0");
  if (layout < 0 || layout > LBM_LAYOUT_POINTER_TILE) return fail(LBM_EINVAL, "unknown layout %d", layout);
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(LBM_EINVAL, "device %d not present", device);
  DeviceGuard dg(device);
  constexpr int kChunk = 256;  // the reference's TILE_NODES (16 x 16)
  const long long n = block_bytes / 8 / kChunk * kChunk;
  double *src = nullptr, *dst = nullptr;
  uint8_t* mask = nullptr;
  long long* base = nullptr;
  unsigned long long* bad = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = 0;
  cudaError_t e = cudaMalloc(&src, n * 8);
  if (e == cudaSuccess) e = cudaMalloc(&dst, n * 8);
  if (e == cudaSuccess) e = cudaMalloc(&bad, 8);
  if (e == cudaSuccess && layout == LBM_LAYOUT_BITMASK_NODE) e = cudaMalloc(&mask, n);
  if (e == cudaSuccess && layout == LBM_LAYOUT_POINTER_TILE) e = cudaMalloc(&base, n / kChunk * 8);
  if (e != cudaSuccess) {
    cudaGetLastError();
    rc = fail(LBM_ENOMEM, "copy bench: cannot allocate 2 x %lld byte blocks", n * 8);
  } else {
    k_iota<<<1184, 256>>>(src, n);
    cudaMemset(dst, 0, n * 8);
    cudaMemset(bad, 0, 8);
    if (mask) cudaMemset(mask, 1, n);
    if (base) {
      std::vector<long long> hb(n / kChunk);
      for (size_t c = 0; c < hb.size(); ++c) hb[c] = (long long)c * kChunk;
      cudaMemcpy(base, hb.data(), hb.size() * 8, cudaMemcpyHostToDevice);
    }
    auto run = [&]() {
      if (layout == LBM_LAYOUT_DENSE)
        k_copy_dense<<<(unsigned)((n / 2 + 1023) / 1024), 256>>>((const double2*)src, (double2*)dst, n / 2);
      else if (layout == LBM_LAYOUT_BITMASK_NODE)
        k_copy_masked<<<148 * 8, 256>>>(src, dst, mask, n);
      else
        k_copy_chunked<<<(unsigned)(n / kChunk), kChunk, 0>>>(src, dst, base, kChunk);
    };
    for (int k = 0; k < warmup; ++k) run();
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int k = 0; k < repetitions; ++k) run();
    cudaEventRecord(e1);
    e = cudaEventSynchronize(e1);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long nbad = 0;
    if (e == cudaSuccess) {
      k_count_diff<<<1184, 256>>>(src, dst, n, bad);
      e = cudaMemcpy(&nbad, bad, 8, cudaMemcpyDeviceToHost);
    }
    if (e != cudaSuccess)
      rc = fail(LBM_ECUDA, "copy bench: %s", cudaGetErrorString(e));
    else if (nbad)
      rc = fail(LBM_ESTATE, "copy benchmark produced a corrupted destination (%llu elements)", nbad);
    else
      *bytes_per_s = 2.0 * (double)n * 8.0 * repetitions / (ms / 1e3);
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  for (void* p : {(void*)src, (void*)dst, (void*)mask, (void*)base, (void*)bad})
    if (p) cudaFree(p);
  return rc;
}

int lbm_create(const lbm_desc* desc, lbm_t** out) {
  if (!desc || !out) return fail(LBM_EINVAL, "desc/out is NULL");
  const lbm_desc& d = *desc;
  if (d.nx <= 0 || d.ny <= 0 || d.nz <= 0)
    return fail(LBM_EINVAL, "dims must be positive, got (%d, %d, %d)", d.nx, d.ny, d.nz);
  if (d.dtype != LBM_F32 && d.dtype != LBM_F64) return fail(LBM_EINVAL, "dtype must be LBM_F32 or LBM_F64");
  if (d.layout < 0 || d.layout > LBM_LAYOUT_POINTER_TILE) return fail(LBM_EINVAL, "unknown layout %d", d.layout);
  if (!(d.omega > 0.0 && d.omega < 2.0)) return fail(LBM_EINVAL, "omega must lie in (0, 2), got %g", d.omega);
  if (d.scheme != LBM_SCHEME_AB && d.scheme != LBM_SCHEME_AA) return fail(LBM_EINVAL, "unknown scheme %d", d.scheme);
  const int nzg = d.nz_global > 0 ? d.nz_global : d.nz;
  if (d.z0 < 0 || d.z0 + d.nz > nzg) return fail(LBM_EINVAL, "slab [%d, %d) outside nz_global %d", d.z0, d.z0 + d.nz, nzg);
  if (!is_tiled(d.layout) && (long long)(d.nz + 2) * d.ny * ((d.nx + 31) / 32 * 32) + 64 >= (1LL << 32))
    return fail(LBM_EINVAL, "dense slab of %d x %d x %d nodes exceeds 2^32 slots; split it into z-slabs", d.nx, d.ny, d.nz);
  if (is_tiled(d.layout)) {
    for (int a = 0; a < 3; ++a) {
      const int e = d.tile[a];
      if (e < 1 || (e & (e - 1))) return fail(LBM_EINVAL, "tile edges must be powers of two, got %d", e);
    }
    if (d.tile[0] * d.tile[1] * d.tile[2] > 512 || d.tile[0] * d.tile[1] * d.tile[2] < 32)
      return fail(LBM_EINVAL, "tile must hold 32..512 nodes");
    const int n3[3] = {d.nx, d.ny, d.nz};
    for (int a = 0; a < 3; ++a)
      if (d.periodic[a] && n3[a] % d.tile[a])
        return fail(LBM_EINVAL, "periodic axis %d needs extent %d divisible by the tile edge %d", a, n3[a], d.tile[a]);
  }
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (d.device < 0 || d.device >= ndev) return fail(LBM_EINVAL, "device %d not present (%d devices)", d.device, ndev);
  DeviceGuard dg(d.device);
  lbm_handle* h = new lbm_handle();
  h->d = d;
  h->d.nz_global = nzg;
  h->esize = d.dtype == LBM_F32 ? 4 : 8;
  Geo& g = h->g;
  g.nx = d.nx;
  g.ny = d.ny;
  g.nz = d.nz;
  g.px = d.periodic[0] != 0;
  g.py = d.periodic[1] != 0;
  g.pzw = (d.periodic[2] != 0) && (nzg == d.nz);
  g.tiled = is_tiled(d.layout);
  g.aa = d.scheme == LBM_SCHEME_AA;
  {
    const char* zf = getenv("LBM_ZERO_FILL");  // A/B switch for the sector-completion stores
    g.zero_fill = (zf && zf[0] == '0') ? 0 : 1;
    const char* sv = getenv("LBM_STEP_VARIANT");
    h->variant = sv ? atoi(sv) : 0;
    h->variant_set = sv != nullptr;
    const char* ub = getenv("LBM_UBITS");
    h->use_ubits = !(ub && ub[0] == '0');
    const char* gv = getenv("LBM_GRAPH");
    h->use_graph = !(gv && gv[0] == '0');
  }
  h->n_nodes = (long long)d.nx * d.ny * d.nz;
  if (!g.tiled) {
    g.nxp = (d.nx + 31) / 32 * 32;
    g.plane = (long long)g.ny * g.nxp;
    h->n_slots = (long long)(g.nz + 2) * g.plane;
    g.ps = (h->n_slots + 63) / 64 * 64;
    h->nflags = (long long)g.nz * g.plane;
  } else {
    g.ex = d.tile[0];
    g.ey = d.tile[1];
    g.ez = d.tile[2];
    g.lex = ilog2(g.ex);
    g.ley = ilog2(g.ey);
    g.lez = ilog2(g.ez);
    {
      // one 32-B sector per brick: 2x2x2 fp32, 2x2x1 fp64 (LBM_BRICK=0: x-rows)
      const char* bv = getenv("LBM_BRICK");
      const bool rows = bv && bv[0] == '0';
      const int want = d.dtype == LBM_F32 ? 3 : 2;  // log2(nodes per sector)
      int b[3] = {0, 0, 0}, left = want;
      if (rows) {  // x first, then y, z: a brick still fills one sector
        b[0] = want < g.lex ? want : g.lex;
        left = want - b[0];
        b[1] = left < g.ley ? left : g.ley;
        b[2] = want - b[0] - b[1];
      } else {
        for (int a = 0; left > 0 && a < 3 * 4; ++a) {
          const int ax = a % 3, lim = ax == 0 ? g.lex : (ax == 1 ? g.ley : g.lez);
          if (b[ax] < lim) { ++b[ax]; --left; }
        }
      }
      g.lbx = b[0];
      g.lby = b[1];
      g.lbz = b[2];
    }
    g.gx = (d.nx + g.ex - 1) / g.ex;
    g.gy = (d.ny + g.ey - 1) / g.ey;
    g.gz = (d.nz + g.ez - 1) / g.ez;
    g.tn = g.ex * g.ey * g.ez;
    g.ltn = ilog2(g.tn);
    g.nxp = d.nx;
    h->ntiles_grid = (long long)g.gx * g.gy * g.gz;
  }
  cudaError_t e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&h->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&h->ev1);
  if (e == cudaSuccess) e = cudaMalloc(&h->scratch, 4096 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&h->uscratch, 4 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&h->sync, 4 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(h->sync, 0, 4 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&h->herr, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(h->herr, 0, sizeof(int));
  if (e != cudaSuccess) {
    lbm_destroy(h);
    return fail(LBM_ECUDA, "stream/event setup: %s", cudaGetErrorString(e));
  }
  *out = h;
  return 0;
}

void lbm_destroy(lbm_t* h) {
  if (!h) return;
  DeviceGuard dg(h->d.device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (lbm_handle::Peer* pr : {&h->lo, &h->hi}) {
    if (pr->on && pr->ipc) {
      cudaIpcCloseMemHandle(pr->f[0]);
      if (pr->f[1] != pr->f[0]) cudaIpcCloseMemHandle(pr->f[1]);
      cudaIpcCloseMemHandle(pr->sync);
      if (pr->rank) cudaIpcCloseMemHandle(pr->rank);
    }
    pr->on = false;
  }
  free_geometry(h);
  dev_free(h->scratch);
  dev_free(h->uscratch);
  dev_free(h->sync);
  dev_free(h->herr);
  for (int b = 0; b < 2; ++b) {
    release_pinned(h->pin[b], h->pin_bytes);
    if (h->evc[b]) cudaEventDestroy(h->evc[b]);
  }
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

// LBM_TIMING=1: phase times of lbm_set_geometry on stderr (device synchronised)
struct PhaseTimer {
  bool on = false;
  cudaStream_t st = nullptr;
  std::chrono::steady_clock::time_point t0;
  explicit PhaseTimer(cudaStream_t s) : st(s) {
    const char* v = getenv("LBM_TIMING");
    on = v && v[0] == '1';
    t0 = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[lbm timing] %-28s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

int lbm_set_geometry(lbm_t* h, const uint8_t* type, const uint8_t* orient, const int32_t* bc_index,
                     const uint8_t* ghost_lo, const uint8_t* ghost_hi, const uint8_t* bc_kind,
                     const double* bc_vel, const double* bc_rho, int32_t nb) {
  NvtxRange nv("lbm_set_geometry");
  if (!h || !type || !orient || !bc_index) return fail(LBM_EINVAL, "NULL geometry array");
  if (nb < 0 || nb > 255) return fail(LBM_EINVAL, "boundary table holds %d entries; at most 255 supported", nb);
  if (nb > 0 && (!bc_kind || !bc_vel || !bc_rho)) return fail(LBM_EINVAL, "NULL boundary table");
  if (h->lo.on || h->hi.on)
    return fail(LBM_ESTATE, "z-slab is connected to its neighbours (they map its buffers): "
                            "destroy the slab handles instead of replacing the geometry");
  DeviceGuard dg(h->d.device);
  CK(cudaStreamSynchronize(h->stream));
  free_geometry(h);
  Geo& g = h->g;
  const long long N = h->n_nodes;
  const long long plane_nodes = (long long)g.nx * g.ny;
  int rc = 0;
  uint8_t *dtype_ = nullptr, *dorient = nullptr, *dglo = nullptr, *dghi = nullptr;  // dtype_: type | orient << 3
  uint8_t* dbc = nullptr;  // bc index byte
  int herr_host = 0;
  int* derr = nullptr;
  int *keep = nullptr, *scan = nullptr;
  void* cub_tmp = nullptr;
  const int nbt = nb > 0 ? nb : 1;
  PhaseTimer pt(h->stream);
  // temporaries
  keep_pool(h->d.device);
  if ((rc = tmp_alloc(h, &dtype_, N)) || (rc = tmp_alloc(h, &dbc, N)) || (rc = tmp_alloc(h, &derr, 16)))
    goto done;
  pt.mark("alloc temporaries");
  if ((rc = upload_descriptors(h, dtype_, dbc, type, orient, bc_index, N, nb, &herr_host))) goto done;
  pt.mark("upload descriptors (packed)");
  if (herr_host & 1) { rc = fail(LBM_EINVAL, "node type or orientation out of range"); goto done; }
  if (herr_host & 2) { rc = fail(LBM_EINVAL, "velocity/pressure node without a valid bc_index or orientation"); goto done; }
  CK(cudaMemsetAsync(derr, 0, 16, h->stream));
  CK(cudaMemsetAsync(h->uscratch, 0, 4 * sizeof(unsigned long long), h->stream));
  h->has_glo = ghost_lo != nullptr;  // z-slab: links cross z = -1 / z = nz into a neighbour
  h->has_ghi = ghost_hi != nullptr;
  if (ghost_lo) {
    if ((rc = tmp_alloc(h, &dglo, plane_nodes))) goto done;
    CK(cudaMemcpyAsync(dglo, ghost_lo, plane_nodes, cudaMemcpyHostToDevice, h->stream));
  } else if (g.pzw) {
    dglo = nullptr;  // wrap handled below
  }
  if (ghost_hi) {
    if ((rc = tmp_alloc(h, &dghi, plane_nodes))) goto done;
    CK(cudaMemcpyAsync(dghi, ghost_hi, plane_nodes, cudaMemcpyHostToDevice, h->stream));
  }
  {
    // whole-domain periodic z: the ghost planes are the wrapped planes
    const uint8_t* glo = dglo ? dglo : (g.pzw ? dtype_ + (long long)(g.nz - 1) * plane_nodes : nullptr);
    const uint8_t* ghi = dghi ? dghi : (g.pzw ? dtype_ : nullptr);
    // boundary tables (float64 for init, storage type for the step)
    if ((rc = dev_alloc(h, &h->bckind64, nbt)) || (rc = dev_alloc(h, &h->bcv64, nbt * 3 * 8)) ||
        (rc = dev_alloc(h, &h->bcr64, nbt * 8)) || (rc = dev_alloc(h, (char**)&h->bcv, nbt * 3 * h->esize)) ||
        (rc = dev_alloc(h, (char**)&h->bcr, nbt * h->esize)))
      goto done;
    {
      std::vector<uint8_t> kk(nbt, 0);
      std::vector<double> vv(nbt * 3, 0.0), rr(nbt, 0.0);
      for (int b = 0; b < nb; ++b) {
        kk[b] = bc_kind[b];
        for (int c = 0; c < 3; ++c) vv[3 * b + c] = bc_vel[3 * b + c];
        rr[b] = bc_rho[b];
      }
      CK(scopy(h, h->bckind64, kk.data(), nbt, cudaMemcpyHostToDevice));
      CK(scopy(h, h->bcv64, vv.data(), nbt * 3 * 8, cudaMemcpyHostToDevice));
      CK(scopy(h, h->bcr64, rr.data(), nbt * 8, cudaMemcpyHostToDevice));
      if (h->esize == 4) {
        std::vector<float> vf(nbt * 3), rf(nbt);
        for (int k = 0; k < nbt * 3; ++k) vf[k] = (float)vv[k];
        for (int k = 0; k < nbt; ++k) rf[k] = (float)rr[k];
        CK(scopy(h, h->bcv, vf.data(), nbt * 3 * 4, cudaMemcpyHostToDevice));
        CK(scopy(h, h->bcr, rf.data(), nbt * 4, cudaMemcpyHostToDevice));
      } else {
        CK(scopy(h, h->bcv, vv.data(), nbt * 3 * 8, cudaMemcpyHostToDevice));
        CK(scopy(h, h->bcr, rr.data(), nbt * 8, cudaMemcpyHostToDevice));
      }
    }
    if (!g.tiled) {
      if ((rc = dev_alloc(h, &h->flags, h->nflags * 4))) goto done;
      dim3 grid((g.nxp + 127) / 128, g.ny, g.nz);
      k_flags_dense<<<grid, 128, 0, h->stream>>>(h->flags, dtype_, dbc, glo, ghi, g, h->uscratch);
      CKL();
      const long long nwords = (h->nflags + 1023) / 1024;
      if ((rc = dev_alloc(h, &h->ubits, nwords * 4))) goto done;
      CK(cudaMemsetAsync(h->ubits, 0, nwords * 4, h->stream));
      if (h->use_ubits) {
        k_uniform_bits<<<(unsigned)((h->nflags + 255) / 256), 256, 0, h->stream>>>(h->ubits, h->flags, h->nflags);
        CKL();
      }
      {
        std::vector<uint32_t> hb(nwords);
        CK(cudaMemcpyAsync(hb.data(), h->ubits, nwords * 4, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        long long uni = 0;
        for (uint32_t v : hb) uni += __builtin_popcount(v);
        // the step reads the bitmap plus the flag words of non-uniform chunks
        h->meta_bytes = nwords * 4 + (h->nflags - 32 * uni) * 4;
      }
    } else {
      const long long G = h->ntiles_grid;
      if ((rc = dev_alloc(h, &h->rank, G * 4)) || (rc = tmp_alloc(h, &keep, G * 4)) ||
          (rc = tmp_alloc(h, &scan, G * 4)))
        goto done;
      const int keep_all = h->d.layout == LBM_LAYOUT_TILE;
      pt.mark("upload descriptors");
      k_tile_keep<<<(unsigned)((G * 32 + 255) / 256), 256, 0, h->stream>>>(keep, dtype_, g, keep_all, G);
      CKL();
      size_t tmp_bytes = 0;
      if (G > 0x7fffffffLL) { rc = fail(LBM_EINVAL, "too many tiles"); goto done; }
      CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, keep, scan, (int)G, h->stream));
      if ((rc = tmp_alloc(h, (char**)&cub_tmp, tmp_bytes))) goto done;
      CK(cub::DeviceScan::ExclusiveSum(cub_tmp, tmp_bytes, keep, scan, (int)G, h->stream));
      int last_scan = 0, last_keep = 0;
      CK(cudaMemcpyAsync(&last_scan, scan + G - 1, 4, cudaMemcpyDeviceToHost, h->stream));
      CK(cudaMemcpyAsync(&last_keep, keep + G - 1, 4, cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      const long long T = (long long)last_scan + last_keep;
      if (T * g.tn >= (1LL << 31)) { rc = fail(LBM_EINVAL, "%lld kept tiles exceed 2^31 slots", T); goto done; }
      h->n_tiles = T;
      if ((rc = dev_alloc(h, &h->tiles, (T > 0 ? T : 1) * 3 * 4)) ||
          (rc = dev_alloc(h, &h->nbr27, (T > 0 ? T : 1) * 27 * 4)))
        goto done;
      pt.mark("tile keep + scan");
      k_tile_compact<<<(unsigned)((G + 255) / 256), 256, 0, h->stream>>>(h->rank, keep, scan, h->tiles, g, G);
      CKL();
      if (T > 0) {
        k_tile_nbr<<<(unsigned)((T * 27 + 255) / 256), 256, 0, h->stream>>>(h->nbr27, h->tiles, h->rank, g, T);
        CKL();
      }
      h->n_slots = T * g.tn;
      g.ps = h->n_slots;  // AoSoA: 19 * ps elements = T tiles x 19 blocks
      h->nflags = h->n_slots;
      if ((rc = dev_alloc(h, &h->flags, (h->nflags > 0 ? h->nflags : 1) * 4))) goto done;
      if (h->nflags > 0) {
        pt.mark("compact + nbr27 + order");
        k_flags_tile<<<(unsigned)((h->nflags + 255) / 256), 256, 0, h->stream>>>(
            h->flags, h->tiles, dtype_, dbc, glo, ghi, g, h->nflags, h->uscratch);
        CKL();
      }
      if ((rc = dev_alloc(h, &h->bmask, (T > 0 ? T : 1) * 32))) goto done;
      CK(cudaMemsetAsync(h->bmask, 0, (T > 0 ? T : 1) * 32, h->stream));
      const int bn = 1 << (g.lbx + g.lby + g.lbz);
      const long long nbricks = h->nflags / bn;
      if (nbricks > 0) {
        k_brick_mask<<<(unsigned)((nbricks + 255) / 256), 256, 0, h->stream>>>(h->bmask, h->flags, g, nbricks);
        CKL();
      }
      if (!h->use_ubits) CK(cudaMemset2DAsync(h->bmask + 4, 32, 0, 16, (T > 0 ? T : 1), h->stream));
      {
        pt.mark("flags + brick masks");
        std::vector<uint32_t> hb((T > 0 ? T : 1) * 8);
        CK(cudaMemcpyAsync(hb.data(), h->bmask, hb.size() * 4, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        long long live = 0, uni = 0;
        for (size_t k = 0; k < hb.size(); ++k) (k % 8 < 4 ? live : uni) += __builtin_popcount(hb[k]);
        // warp work list: groups of (32 / bricksize) live bricks per tile, each
        // item decoded on the host into {tile, brick byte per lane group (two
        // words), uniform bits | count << 8}, so a warp reaches its data loads
        // after one dependent load instead of walking the brick masks
        {
          const int per = 32 / bn;  // 4 (fp32 2x2x2 bricks) or 8 (fp64 2x2x1)
          // an item packs at most 8 brick bytes and a 4-bit count; smaller
          // bricks (LBM_BRICK=0 with a tile x-edge under one sector) run the
          // CTA-per-tile kernels instead
          h->wlist_ok = per <= 8;
          std::vector<uint32_t> it;
          it.reserve((size_t)(live / per + T) * 4);
          for (long long k2 = 0; h->wlist_ok && k2 < T; ++k2) {
            const long long t = k2;
            uint32_t rec[4] = {(uint32_t)t, 0u, 0u, 0u};
            int k = 0;
            for (int q = 0; q < 4; ++q) {
              for (uint32_t mq = hb[8 * t + q]; mq; mq &= mq - 1) {
                const int b = q * 32 + __builtin_ctz(mq);
                rec[1 + k / 4] |= (uint32_t)b << (8 * (k & 3));
                if ((hb[8 * t + 4 + q] >> (b & 31)) & 1u) rec[3] |= 1u << k;
                if (++k == per) {
                  rec[3] |= (uint32_t)k << 8;
                  it.insert(it.end(), rec, rec + 4);
                  rec[1] = rec[2] = rec[3] = 0u;
                  k = 0;
                }
              }
            }
            if (k) {
              rec[3] |= (uint32_t)k << 8;
              it.insert(it.end(), rec, rec + 4);
            }
          }
          // z-slabs: items of the first / last tile plane first (they hold the
          // ghost exchange), so the step can signal its neighbours before the
          // interior items run
          h->n_items_b = 0;
          if ((h->has_glo || h->has_ghi) && !it.empty() && T > 0) {
            std::vector<int> tz((size_t)T * 3);
            CK(scopy(h, tz.data(), h->tiles, (size_t)T * 12, cudaMemcpyDeviceToHost));
            std::vector<uint32_t> bnd, inner;
            for (size_t k = 0; k < it.size(); k += 4) {
              const int z3 = tz[3 * (size_t)it[k] + 2];
              auto& dst = (z3 == 0 || z3 == g.gz - 1) ? bnd : inner;
              dst.insert(dst.end(), it.begin() + k, it.begin() + k + 4);
            }
            h->n_items_b = (int)(bnd.size() / 4);
            bnd.insert(bnd.end(), inner.begin(), inner.end());
            it.swap(bnd);
          }
          pt.mark("brick masks to host + work list");
          h->n_items = (int)(it.size() / 4);
          if ((rc = dev_alloc(h, &h->items, (it.size() ? it.size() : 4) * 4))) goto done;
          if (!it.empty()) CK(scopy(h, h->items, it.data(), it.size() * 4, cudaMemcpyHostToDevice));
        }
        // the warp work list is the default for every tile shape unless the
        // kept tiles are (almost) all live bricks: round 2 measured it ahead
        // of or level with one CTA per tile at every porosity and tile shape
        // (profiles/tile_sweep_r02ag.txt; round 1 had enabled it only for
        // 512-node tiles below live fraction 0.85)
        const double live_frac = T > 0 ? (double)live / ((double)T * (g.tn / bn)) : 1.0;
        h->auto_wlist = h->wlist_ok && live_frac < 0.99;
        h->live_frac = live_frac;
        // per tile: nbr27 + brick masks; per live, non-uniform brick: its flag
        // words; the work list when it is used
        h->meta_bytes = T * (27 * 4 + 32) + (live - uni) * bn * 4 +
                        (h->auto_wlist ? (long long)h->n_items * 16 : 0);
      }
      h->sm.rank = h->rank;
      {
        // per-slot neighbour table for the tile kernels (TileUpLUT): in-tile
        // slot deltas per axis (the slot order is separable over x / y / z)
        auto P = [](int l) { return l; };
        std::vector<unsigned long long> lt(2 * (size_t)g.tn);
        for (int l = 0; l < g.tn; ++l) {
          int lx, ly, lz;
          brick_inv(g, l, lx, ly, lz);
          const int e[3] = {g.ex, g.ey, g.ez}, c[3] = {lx, ly, lz};
          int mag[6];
          unsigned cross = 0;
          for (int a = 0; a < 3; ++a) {
            auto br = [&](int v) { return a == 0 ? brick_x(g, v) : (a == 1 ? brick_y(g, v) : brick_z(g, v)); };
            const int own = P(br(c[a]));
            const bool cm = c[a] == 0, cp = c[a] == e[a] - 1;
            const int mm = P(br(cm ? e[a] - 1 : c[a] - 1)) - own, mp = P(br(cp ? 0 : c[a] + 1)) - own;
            mag[2 * a] = mm < 0 ? -mm : mm;
            mag[2 * a + 1] = mp < 0 ? -mp : mp;
            cross |= (cm ? 1u : 0u) << (2 * a);
            cross |= (cp ? 1u : 0u) << (2 * a + 1);
          }
          unsigned long long x = 0, y = 0;
          for (int k = 0; k < 4; ++k) x |= (unsigned long long)mag[k] << (14 * k);
          x |= (unsigned long long)cross << 56;
          y = (unsigned long long)mag[4] | (unsigned long long)mag[5] << 14 | (unsigned long long)P(l) << 32;
          lt[2 * l] = x;
          lt[2 * l + 1] = y;
        }
        if ((rc = dev_alloc(h, &h->lut, lt.size() * 8))) goto done;
        CK(scopy(h, h->lut, lt.data(), lt.size() * 8, cudaMemcpyHostToDevice));
      }
      // z-slab ghost planes (AB tile layouts keep them outside the tile
      // storage; A-A tile slabs reach into the neighbour directly)
      if ((h->has_glo || h->has_ghi) && !g.aa) {
        const size_t gb = (size_t)10 * plane_nodes * h->esize;
        if ((rc = dev_alloc(h, (char**)&h->gh[0], gb)) || (rc = dev_alloc(h, (char**)&h->gh[1], gb))) goto done;
        CK(cudaMemsetAsync(h->gh[0], 0, gb, h->stream));
        CK(cudaMemsetAsync(h->gh[1], 0, gb, h->stream));
      }
    }
    int herr = 0;
    unsigned long long nons = 0;
    CK(cudaMemcpyAsync(&herr, derr, 4, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(&nons, h->uscratch, 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (herr & 1) { rc = fail(LBM_EINVAL, "node type or orientation out of range"); goto done; }
    if (herr & 2) { rc = fail(LBM_EINVAL, "velocity/pressure node without a valid bc_index or orientation"); goto done; }
    h->n_nonsolid = (long long)nons;
    h->nb = nb;
    // release the descriptor temporaries before the PDF buffers claim HBM
    // (a 2^31-node domain needs every byte: 163 GB AA PDFs + 8.6 GB flags)
    for (void** p : {(void**)&dtype_, (void**)&dorient, (void**)&dbc, (void**)&dglo, (void**)&dghi,
                     (void**)&keep, (void**)&scan, (void**)&cub_tmp}) {
      tmp_free(h, *p);
      *p = nullptr;
    }
    pt.mark("geometry done");
    // PDF buffers
    const size_t fbytes = (size_t)(buf_elems(h) > 0 ? buf_elems(h) : 64) * h->esize;
    {
      // a domain that fills HBM needs the pool's cached temporaries back
      size_t fr = 0, tot = 0;
      CK(cudaStreamSynchronize(h->stream));
      cudaMemGetInfo(&fr, &tot);
      if (fr < (g.aa ? 1 : 2) * fbytes + (1ull << 30)) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, h->d.device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
        cudaGetLastError();
      }
    }
    if ((rc = dev_alloc(h, (char**)&h->f[0], fbytes))) goto done;
    if (!g.aa && (rc = dev_alloc(h, (char**)&h->f[1], fbytes))) goto done;  // AA: one buffer
    CK(cudaMemsetAsync(h->f[0], 0, fbytes, h->stream));
    if (h->f[1]) CK(cudaMemsetAsync(h->f[1], 0, fbytes, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    pt.mark("PDF buffers alloc + zero");
    h->geometry = true;
    h->parity = 0;
    h->step_count = h->visited_total = 0;
  }
done:
  {
    cudaStreamSynchronize(h->stream);
    tmp_free(h, dtype_);
    tmp_free(h, dorient);
    tmp_free(h, dbc);
    tmp_free(h, dglo);
    tmp_free(h, dghi);
    tmp_free(h, derr);
    tmp_free(h, keep);
    tmp_free(h, scan);
    tmp_free(h, cub_tmp);
    // recompute resident bytes (temporaries released)
    if (h->geometry) {
      long long b = (h->g.aa ? 1LL : 2LL) * (buf_elems(h) > 0 ? buf_elems(h) : 64) * h->esize + h->nflags * 4;
      if (h->g.tiled) b += h->ntiles_grid * 4 + h->n_tiles * (30 + 8) * 4;
      if (h->gh[0]) b += 2LL * 10 * h->g.nx * h->g.ny * h->esize;
      h->device_bytes = b;
    }
  }
  if (rc) free_geometry(h);
  return rc;
}

int lbm_init_equilibrium(lbm_t* h, const double* rho, const double* ux, const double* uy,
                         const double* uz, double rho0, double ux0, double uy0, double uz0) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  if (!h->geometry) return fail(LBM_ESTATE, "lbm_set_geometry must run before lbm_init_equilibrium");
  DeviceGuard dg(h->d.device);
  const Geo& g = h->g;
  const long long N = h->n_nodes;
  const double* src[4] = {rho, ux, uy, uz};
  double* dev[4] = {nullptr, nullptr, nullptr, nullptr};
  int rc = 0;
  for (int k = 0; k < 4 && !rc; ++k) {
    if (!src[k]) continue;
    cudaError_t e = cudaMalloc(&dev[k], N * 8);
    if (e != cudaSuccess) {
      rc = fail(LBM_ENOMEM, "init field upload: %s", cudaGetErrorString(e));
      break;
    }
    e = cudaMemcpyAsync(dev[k], src[k], N * 8, cudaMemcpyHostToDevice, h->stream);
    if (e != cudaSuccess) rc = fail(LBM_ECUDA, "init upload: %s", cudaGetErrorString(e));
  }
  if (!rc) {
    const size_t fbytes = (size_t)buf_elems(h) * h->esize;
    cudaMemsetAsync(h->f[0], 0, fbytes, h->stream);
    if (h->f[1]) cudaMemsetAsync(h->f[1], 0, fbytes, h->stream);
    h->parity = 0;
    const int bx = 128;
    if (h->esize == 4)
      k_init<float><<<node_grid(g, bx), bx, 0, h->stream>>>((float*)h->f[0], h->flags, h->sm, g, dev[0], dev[1],
                                                            dev[2], dev[3], rho0, ux0, uy0, uz0, h->bckind64,
                                                            h->bcv64, h->bcr64, h->nb);
    else
      k_init<double><<<node_grid(g, bx), bx, 0, h->stream>>>((double*)h->f[0], h->flags, h->sm, g, dev[0], dev[1],
                                                             dev[2], dev[3], rho0, ux0, uy0, uz0, h->bckind64,
                                                             h->bcv64, h->bcr64, h->nb);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) rc = fail(LBM_ECUDA, "k_init: %s", cudaGetErrorString(e));
  }
  for (int k = 0; k < 4; ++k) dev_free(dev[k]);
  if (rc) return rc;
  h->initialized = true;
  h->halo_dirty = true;
  h->step_count = h->visited_total = 0;
  return 0;
}

int lbm_set_omega(lbm_t* h, double omega) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  if (!(omega > 0.0 && omega < 2.0)) return fail(LBM_EINVAL, "omega must lie in (0, 2), got %g", omega);
  h->d.omega = omega;
  drop_graphs(h);
  return 0;
}

// kGraphSteps steps starting at parity p0, captured into h->graph[p0] once
static int capture_graph(lbm_handle* h, int p0) {
  cudaGraphExec_t& ge = h->graph[p0];
  if (ge) return 0;
  const bool halo = halo_on(h);
  const int keep = h->parity;
  const long long l0 = h->launches;
  h->parity = p0;
  cudaGraph_t gr = nullptr;
  CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  for (int k = 0; k < kGraphSteps; ++k) {
    void* post = h->g.aa ? h->f[0] : h->f[1 - h->parity];
    if (h->esize == 4) {
      if (halo) slab_step<float>(h, pre_buf(h), post); else launch_step<float>(h, pre_buf(h), post);
    } else {
      if (halo) slab_step<double>(h, pre_buf(h), post); else launch_step<double>(h, pre_buf(h), post);
    }
    h->parity ^= 1;
  }
  CK(cudaStreamEndCapture(h->stream, &gr));
  h->parity = keep;
  h->graph_launches = h->launches - l0;
  h->launches = l0;
  cudaError_t e = cudaGraphInstantiate(&ge, gr, 0);
  cudaGraphDestroy(gr);
  if (e == cudaSuccess) e = cudaGraphUpload(ge, h->stream);
  if (e != cudaSuccess) return fail(LBM_ECUDA, "cuda graph: %s", cudaGetErrorString(e));
  return 0;
}

int lbm_step_async(lbm_t* h, int64_t n) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  NvtxRange nv("lbm_step");
  if (n < 0) return fail(LBM_EINVAL, "n_steps must be >= 0, got %lld", (long long)n);
  if (!h->initialized) return fail(LBM_ESTATE, "initialize() must run before stepping");
  if (n > 0 && ((h->has_glo && !h->lo.on) || (h->has_ghi && !h->hi.on)))
    return fail(LBM_ESTATE, "z-slab has a ghost plane on its %s side but no neighbour is connected "
                            "(lbm_halo_connect)", (h->has_glo && !h->lo.on) ? "lower" : "upper");
  DeviceGuard dg(h->d.device);
  const bool halo = halo_on(h);
  if (halo && h->halo_dirty && n > 0) {
    // ghost planes of `pre` after initialize / set_pdf: push, then signal
    // (A-A reads the neighbours' planes directly: signal only)
    if (!h->g.aa) {
      if (h->esize == 4) halo_push<float>(h); else halo_push<double>(h);
    }
    halo_signal(h);
    h->halo_dirty = false;
  }
  CK(cudaEventRecord(h->ev0, h->stream));
  // launch-bound small domains: replay a captured CUDA graph of kGraphSteps
  // steps (an even count, so it starts and ends on the same parity)
  // z-slabs capture their wait / boundary / signal / interior sequence too
  // (the epochs live on the device; connected slabs capture at connect time)
  if (h->use_graph && n >= kGraphSteps) {
    if (int rc = capture_graph(h, h->parity)) return rc;
    cudaGraphExec_t& ge = h->graph[h->parity];
    while (n >= kGraphSteps) {
      CK(cudaGraphLaunch(ge, h->stream));
      h->launches += h->graph_launches;
      n -= kGraphSteps;
      h->step_count += kGraphSteps;
      h->visited_total += kGraphSteps * visits_per_step(h);
    }
  }
  for (int64_t k = 0; k < n; ++k) {
    const void* pre = pre_buf(h);
    void* post = h->g.aa ? h->f[0] : h->f[1 - h->parity];
    // slabs: neighbours pushed my ghosts and finished reading theirs
    if (h->esize == 4) {
      if (halo) slab_step<float>(h, pre, post); else launch_step<float>(h, pre, post);
    } else {
      if (halo) slab_step<double>(h, pre, post); else launch_step<double>(h, pre, post);
    }
    h->parity ^= 1;
  }
  CKL();
  CK(cudaEventRecord(h->ev1, h->stream));
  h->pending = true;
  h->step_count += n;
  h->visited_total += n * visits_per_step(h);
  return 0;
}

int lbm_synchronize(lbm_t* h) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  NvtxRange nv("lbm_synchronize");
  DeviceGuard dg(h->d.device);
  if (!h->pending) return 0;
  h->pending = false;
  CK(cudaEventSynchronize(h->ev1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  h->last_ms = ms;
  if (halo_on(h)) {
    int herr = 0;
    CK(scopy(h, &herr, h->herr, 4, cudaMemcpyDeviceToHost));
    if (herr) return fail(LBM_ENCCL, "halo wait timed out: a neighbouring slab stopped stepping");
  }
  return 0;
}

int lbm_step(lbm_t* h, int64_t n) {
  int rc = lbm_step_async(h, n);
  if (rc) return rc;
  return lbm_synchronize(h);
}

// z-planes per readback chunk: device staging bounded by kStageBytes, so
// readbacks work next to a domain that fills HBM
constexpr long long kStageBytes = 1LL << 30;
int chunk_planes(const lbm_handle* h, long long bytes_per_node) {
  const long long plane = (long long)h->g.nx * h->g.ny * bytes_per_node;
  long long c = kStageBytes / (plane > 0 ? plane : 1);
  if (c < 1) c = 1;
  if (c > h->g.nz) c = h->g.nz;
  if (c > 65535) c = 65535;  // grid z limit
  return (int)c;
}


int lbm_get_macroscopic(lbm_t* h, double* rho, double* ux, double* uy, double* uz) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  NvtxRange nv("lbm_get_macroscopic");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  DeviceGuard dg(h->d.device);
  const Geo g = rb_geo(h);
  const long long pn = (long long)g.nx * g.ny;
  double* outs[4] = {rho, ux, uy, uz};
  int nf = 0, which[4];
  for (int k = 0; k < 4; ++k)
    if (outs[k]) which[nf++] = k;
  if (!nf) return 0;
  // staging chunk: the requested fields back to back, (nf, nzc * pn) doubles
  auto launch = [&](int, int z0, int nzc, char* dev) {
    double* d = (double*)dev;
    const long long C = (long long)nzc * pn;
    double* f[4] = {nullptr, nullptr, nullptr, nullptr};
    for (int j = 0; j < nf; ++j) f[which[j]] = d + j * C;
    const dim3 grid((g.nx + 127) / 128, g.ny, nzc);
    if (h->esize == 4)
      k_macro<float><<<grid, 128, 0, h->stream>>>((const float*)pre_buf(h), h->flags, h->sm, g, z0, f[0], f[1], f[2],
                                                  f[3]);
    else
      k_macro<double><<<grid, 128, 0, h->stream>>>((const double*)pre_buf(h), h->flags, h->sm, g, z0, f[0], f[1],
                                                   f[2], f[3]);
  };
  for (int j = 0; j < nf; ++j) advise_huge(outs[which[j]], (size_t)h->n_nodes * 8);
  auto consume = [&](int, int z0, int nzc, const char* pin) {
    const long long C = (long long)nzc * pn;
    std::vector<std::pair<char*, const char*>> ds;
    std::vector<size_t> n;
    for (int j = 0; j < nf; ++j) {
      ds.emplace_back((char*)(outs[which[j]] + z0 * pn), pin + (size_t)j * C * 8);
      n.push_back((size_t)C * 8);
    }
    par_copy(ds, n);
  };
  return pipelined_d2h(h, 8LL * nf, launch, consume);
}

int lbm_get_macroscopic_box(lbm_t* h, const int32_t* lo, const int32_t* hi, double* rho, double* ux,
                            double* uy, double* uz) {
  if (!h || !lo || !hi) return fail(LBM_EINVAL, "NULL argument");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  const int n3[3] = {h->g.nx, h->g.ny, h->g.nz};
  for (int a = 0; a < 3; ++a)
    if (lo[a] < 0 || hi[a] > n3[a] || lo[a] >= hi[a])
      return fail(LBM_EINVAL, "box [%d, %d) outside axis %d of extent %d", lo[a], hi[a], a, n3[a]);
  DeviceGuard dg(h->d.device);
  const Geo g = rb_geo(h);
  const int bx = hi[0] - lo[0], by = hi[1] - lo[1], bz = hi[2] - lo[2];
  if (by > 65535 || bz > 65535) return fail(LBM_EINVAL, "box too tall for one launch");
  const long long C = (long long)bx * by * bz;
  double* d = nullptr;
  cudaError_t e = cudaMalloc(&d, C * 8 * 4);
  if (e != cudaSuccess) return fail(LBM_ENOMEM, "box readback: %s", cudaGetErrorString(e));
  double* outs[4] = {rho, ux, uy, uz};
  double* f[4];
  for (int k = 0; k < 4; ++k) f[k] = outs[k] ? d + k * C : nullptr;
  const dim3 grid((bx + 127) / 128, by, bz);
  if (h->esize == 4)
    k_macro<float><<<grid, 128, 0, h->stream>>>((const float*)pre_buf(h), h->flags, h->sm, g, lo[2], f[0], f[1], f[2],
                                                f[3], lo[0], lo[1], bx);
  else
    k_macro<double><<<grid, 128, 0, h->stream>>>((const double*)pre_buf(h), h->flags, h->sm, g, lo[2], f[0], f[1],
                                                 f[2], f[3], lo[0], lo[1], bx);
  e = cudaGetLastError();
  for (int k = 0; k < 4 && e == cudaSuccess; ++k)
    if (outs[k]) e = cudaMemcpyAsync(outs[k], d + k * C, C * 8, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  cudaFree(d);
  if (e != cudaSuccess) return fail(LBM_ECUDA, "box readback: %s", cudaGetErrorString(e));
  return 0;
}

int lbm_check_finite(lbm_t* h, int32_t* dir, int32_t* node_xyz) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  DeviceGuard dg(h->d.device);
  const Geo g = rb_geo(h);
  const unsigned long long none = ~0ULL;
  const long long V = g.tiled ? h->n_slots : h->n_nodes;
  CK(cudaMemcpyAsync(h->uscratch, &none, 8, cudaMemcpyHostToDevice, h->stream));
  const int bx = 128;
  if (h->esize == 4)
    k_nonfinite<float><<<node_grid(g, bx), bx, 0, h->stream>>>((const float*)pre_buf(h), h->flags, h->sm, g, V, h->uscratch);
  else
    k_nonfinite<double><<<node_grid(g, bx), bx, 0, h->stream>>>((const double*)pre_buf(h), h->flags, h->sm, g, V, h->uscratch);
  CKL();
  unsigned long long best = 0;
  CK(cudaMemcpyAsync(&best, h->uscratch, 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (best == none) {
    if (dir) *dir = -1;
    return 0;
  }
  const long long i = (long long)(best / (unsigned long long)V);
  const long long v = (long long)(best % (unsigned long long)V);
  int x, y, z;
  if (!g.tiled) {
    x = (int)(v % g.nx);
    y = (int)((v / g.nx) % g.ny);
    z = (int)(v / ((long long)g.nx * g.ny));
  } else {
    const long long t = v / g.tn;
    const int l = (int)(v % g.tn);
    int tc[3];
    CK(scopy(h, tc, h->tiles + 3 * t, 12, cudaMemcpyDeviceToHost));
    int lx, ly, lz;
    brick_inv(g, l, lx, ly, lz);
    x = tc[0] * g.ex + lx;
    y = tc[1] * g.ey + ly;
    z = tc[2] * g.ez + lz;
  }
  if (dir) *dir = (int32_t)i;
  if (node_xyz) {
    node_xyz[0] = x;
    node_xyz[1] = y;
    node_xyz[2] = z;
  }
  return fail(LBM_EDIVERGED, "non-finite distribution at node (%d, %d, %d), direction %lld", x, y, z, i);
}

int lbm_total_mass(lbm_t* h, double* mass) {
  if (!h || !mass) return fail(LBM_EINVAL, "NULL argument");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  DeviceGuard dg(h->d.device);
  const int nblk = 1184;  // 8 x 148 SMs; fixed so the reduction order is fixed
  if (h->esize == 4)
    k_mass_partial<float><<<nblk, 256, 0, h->stream>>>((const float*)pre_buf(h), h->flags, h->sm, h->tiles, rb_geo(h),
                                                       h->nflags, h->scratch);
  else
    k_mass_partial<double><<<nblk, 256, 0, h->stream>>>((const double*)pre_buf(h), h->flags, h->sm, h->tiles, rb_geo(h),
                                                        h->nflags, h->scratch);
  k_mass_final<<<1, 256, 0, h->stream>>>(h->scratch, nblk, h->scratch + nblk);
  CKL();
  CK(cudaMemcpyAsync(mass, h->scratch + nblk, 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return 0;
}

static int pdf_io(lbm_t* h, int which, void* host, bool get) {
  if (!h || !host) return fail(LBM_EINVAL, "NULL argument");
  if (which != 0 && which != 1) return fail(LBM_EINVAL, "which must be 0 (pre) or 1 (post)");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  if (h->g.aa && which != 0) return fail(LBM_EINVAL, "the AA scheme keeps one buffer: there is no post buffer");
  DeviceGuard dg(h->d.device);
  const Geo g = rb_geo(h);
  const long long N = h->n_nodes, pn = (long long)g.nx * g.ny;
  const int es = h->esize;
  const int cz = chunk_planes(h, (long long)Q * es);
  const long long C = pn * cz;
  char* d = nullptr;
  cudaError_t e = cudaMalloc(&d, C * Q * es);
  if (e != cudaSuccess) return fail(LBM_ENOMEM, "pdf staging: %s", cudaGetErrorString(e));
  void* buf = which == 0 ? pre_buf(h) : h->f[1 - h->parity];
  char* hb = (char*)host;
  if (get) {
    cudaFree(d);
    advise_huge(host, (size_t)Q * N * es);
    // pipelined: chunk = (19, nzc * pn) in the storage type
    auto launch = [&](int, int z0, int nzc, char* dev) {
      const dim3 grid((g.nx + 127) / 128, g.ny, nzc);
      if (es == 4)
        k_get_pdf<float><<<grid, 128, 0, h->stream>>>((const float*)buf, h->flags, h->sm, g, z0, (float*)dev);
      else
        k_get_pdf<double><<<grid, 128, 0, h->stream>>>((const double*)buf, h->flags, h->sm, g, z0, (double*)dev);
    };
    auto consume = [&](int, int z0, int nzc, const char* pin) {
      const long long cn = pn * nzc;
      std::vector<std::pair<char*, const char*>> ds;
      std::vector<size_t> n;
      for (int i = 0; i < Q; ++i) {
        ds.emplace_back(hb + (i * N + z0 * pn) * es, pin + (size_t)i * cn * es);
        n.push_back((size_t)cn * es);
      }
      par_copy(ds, n);
    };
    return pipelined_d2h(h, (long long)Q * es, launch, consume);
  }
  // canonical (19, nz, ny, nx): one host block per direction and z chunk
  for (int z0 = 0; z0 < g.nz && e == cudaSuccess; z0 += cz) {
    const int nzc = g.nz - z0 < cz ? g.nz - z0 : cz;
    const long long cn = pn * nzc;
    const dim3 grid((g.nx + 127) / 128, g.ny, nzc);
    if (!get) {
      for (int i = 0; i < Q && e == cudaSuccess; ++i)
        e = cudaMemcpyAsync(d + i * cn * es, hb + (i * N + z0 * pn) * es, cn * es, cudaMemcpyHostToDevice, h->stream);
      if (e != cudaSuccess) break;
      if (es == 4)
        k_set_pdf<float><<<grid, 128, 0, h->stream>>>((float*)buf, h->flags, h->sm, g, z0, (const float*)d);
      else
        k_set_pdf<double><<<grid, 128, 0, h->stream>>>((double*)buf, h->flags, h->sm, g, z0, (const double*)d);
      e = cudaGetLastError();
    } else {
      if (es == 4)
        k_get_pdf<float><<<grid, 128, 0, h->stream>>>((const float*)buf, h->flags, h->sm, g, z0, (float*)d);
      else
        k_get_pdf<double><<<grid, 128, 0, h->stream>>>((const double*)buf, h->flags, h->sm, g, z0, (double*)d);
      e = cudaGetLastError();
      for (int i = 0; i < Q && e == cudaSuccess; ++i)
        e = cudaMemcpyAsync(hb + (i * N + z0 * pn) * es, d + i * cn * es, cn * es, cudaMemcpyDeviceToHost, h->stream);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  }
  cudaFree(d);
  if (e != cudaSuccess) return fail(LBM_ECUDA, "pdf io: %s", cudaGetErrorString(e));
  return 0;
}

int lbm_get_pdf(lbm_t* h, int32_t which, void* out) { return pdf_io(h, which, out, true); }
// A-A z-slab at an odd step count: pre_i of boundary nodes lives in the
// neighbour's memory (the local ghost plane is a read-only mirror)
static int aa_slab_write_guard(const lbm_t* h) {
  if (h && h->g.aa && (h->lo.on || h->hi.on) && h->parity == 1)
    return fail(LBM_ESTATE, "A-A z-slabs accept state writes at even step counts only");
  return 0;
}

int lbm_set_pdf(lbm_t* h, int32_t which, const void* in) {
  if (int rc = aa_slab_write_guard(h)) return rc;
  if (h) h->halo_dirty = true;
  return pdf_io(h, which, (void*)in, false);
}

static int field_io(lbm_t* h, int which, void* host, bool get) {
  if (!h || !host) return fail(LBM_EINVAL, "NULL argument");
  if (which != 0 && which != 1) return fail(LBM_EINVAL, "which must be 0 (pre) or 1 (post)");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  if (h->g.aa && which != 0) return fail(LBM_EINVAL, "the AA scheme keeps one buffer: there is no post buffer");
  DeviceGuard dg(h->d.device);
  const size_t bytes = (size_t)Q * h->g.ps * h->esize;
  if (h->g.aa) {
    // decoded pre buffer in the native slot order, staged on the device
    void* d = nullptr;
    cudaError_t e = cudaMalloc(&d, bytes);
    if (e != cudaSuccess) return fail(LBM_ENOMEM, "field staging: %s", cudaGetErrorString(e));
    const Geo g = rb_geo(h);
    const dim3 grid = node_grid(g, 128);
    if (get) {
      e = cudaMemsetAsync(d, 0, bytes, h->stream);
      if (e == cudaSuccess) {
        if (h->esize == 4)
          k_field_aa<float, true><<<grid, 128, 0, h->stream>>>((float*)h->f[0], h->flags, h->sm, g, (float*)d);
        else
          k_field_aa<double, true><<<grid, 128, 0, h->stream>>>((double*)h->f[0], h->flags, h->sm, g, (double*)d);
        e = cudaGetLastError();
      }
      if (e == cudaSuccess) e = cudaMemcpyAsync(host, d, bytes, cudaMemcpyDeviceToHost, h->stream);
    } else {
      e = cudaMemcpyAsync(d, host, bytes, cudaMemcpyHostToDevice, h->stream);
      if (e == cudaSuccess) {
        if (h->esize == 4)
          k_field_aa<float, false><<<grid, 128, 0, h->stream>>>((float*)h->f[0], h->flags, h->sm, g, (float*)d);
        else
          k_field_aa<double, false><<<grid, 128, 0, h->stream>>>((double*)h->f[0], h->flags, h->sm, g, (double*)d);
        e = cudaGetLastError();
      }
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    cudaFree(d);
    if (e != cudaSuccess) return fail(LBM_ECUDA, "field io: %s", cudaGetErrorString(e));
    return 0;
  }
  void* buf = h->f[which == 0 ? h->parity : 1 - h->parity];
  if (get)
    CK(scopy(h, host, buf, bytes, cudaMemcpyDeviceToHost));
  else
    CK(scopy(h, buf, host, bytes, cudaMemcpyHostToDevice));
  return 0;
}

int lbm_get_field(lbm_t* h, int32_t which, void* out) { return field_io(h, which, out, true); }
int lbm_set_field(lbm_t* h, int32_t which, const void* in) {
  if (int rc = aa_slab_write_guard(h)) return rc;
  if (h) h->halo_dirty = true;
  return field_io(h, which, (void*)in, false);
}

int lbm_get_slot_of(lbm_t* h, int32_t* out) {
  if (!h || !out) return fail(LBM_EINVAL, "NULL argument");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  DeviceGuard dg(h->d.device);
  int* d = nullptr;
  cudaError_t e = cudaMalloc(&d, h->n_nodes * 4);
  if (e != cudaSuccess) return fail(LBM_ENOMEM, "slot_of staging: %s", cudaGetErrorString(e));
  k_slot_of<<<node_grid(h->g, 128), 128, 0, h->stream>>>(h->sm, h->g, d);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, h->n_nodes * 4, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  cudaFree(d);
  if (e != cudaSuccess) return fail(LBM_ECUDA, "slot_of: %s", cudaGetErrorString(e));
  return 0;
}

int lbm_get_flags(lbm_t* h, uint32_t* out) {
  if (!h || !out) return fail(LBM_EINVAL, "NULL argument");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  DeviceGuard dg(h->d.device);
  uint32_t* d = nullptr;
  cudaError_t e = cudaMalloc(&d, h->n_nodes * 4);
  if (e != cudaSuccess) return fail(LBM_ENOMEM, "flags staging: %s", cudaGetErrorString(e));
  k_get_flags<<<node_grid(h->g, 128), 128, 0, h->stream>>>(h->flags, h->sm, h->g, d);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, h->n_nodes * 4, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  cudaFree(d);
  if (e != cudaSuccess) return fail(LBM_ECUDA, "flags: %s", cudaGetErrorString(e));
  return 0;
}

int lbm_get_tile_index(lbm_t* h, int32_t* tiles, int32_t* nbr27, int64_t* n_tiles) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  if (n_tiles) *n_tiles = h->n_tiles;
  if (!h->g.tiled) return 0;
  DeviceGuard dg(h->d.device);
  if (tiles && h->n_tiles) CK(scopy(h, tiles, h->tiles, h->n_tiles * 12, cudaMemcpyDeviceToHost));
  if (nbr27 && h->n_tiles) CK(scopy(h, nbr27, h->nbr27, h->n_tiles * 27 * 4, cudaMemcpyDeviceToHost));
  return 0;
}

int lbm_get_stats(lbm_t* h, lbm_stats* s) {
  if (!h || !s) return fail(LBM_EINVAL, "NULL argument");
  memset(s, 0, sizeof(*s));
  s->n_nodes = h->n_nodes;
  s->n_nonsolid = h->n_nonsolid;
  s->visits_per_step = (h->d.layout == LBM_LAYOUT_DENSE) ? h->n_nodes
                       : (h->d.layout == LBM_LAYOUT_BITMASK_NODE) ? h->n_nonsolid
                                                                   : h->n_slots;
  s->n_slots = h->n_slots;
  s->plane_stride = h->g.ps;
  s->n_tiles = h->n_tiles;
  s->step_count = h->step_count;
  s->visited_nodes_total = h->visited_total;
  s->device_bytes = h->device_bytes;
  s->launches_total = h->launches;
  s->last_step_ms = h->last_ms;
  s->meta_bytes_per_step = h->meta_bytes;
  s->parity = h->parity;
  s->initialized = h->initialized ? 1 : 0;
  s->scheme = h->d.scheme;
  // (z-slab tile handles run the work list with the ghost exchange compiled in)
  s->tile_work_list = h->wlist_ok &&
      ((h->auto_wlist && !h->variant_set) || (h->g.tiled && h->variant == 8)) ? 1 : 0;
  return 0;
}

// ------------------------------------------------------------- halo C-ABI
namespace {
struct HaloBlob {
  uint32_t magic;
  int32_t device, esize, nz, ny, nxp, tiled, aa;
  int32_t ex, ey, ez, gz;   // tile shape and tile-grid depth (tile layouts)
  int64_t pid, ps;
  void* f[2];
  void* sync;
  void* rank;               // tile A-A slabs: the tile rank grid
  cudaIpcMemHandle_t ipc_f[2];
  cudaIpcMemHandle_t ipc_sync;
  cudaIpcMemHandle_t ipc_rank;
};
constexpr uint32_t kHaloMagic = 0x4C424D48u;  // "LBMH"
static_assert(sizeof(HaloBlob) <= LBM_HALO_BLOB_BYTES, "halo blob too large");

int open_peer(lbm_handle* h, const HaloBlob& b, lbm_handle::Peer& pr) {
  if (b.magic != kHaloMagic) return fail(LBM_EINVAL, "not a halo blob");
  if (b.esize != h->esize || b.ny != h->g.ny || b.nxp != h->g.nxp || b.tiled != h->g.tiled ||
      b.aa != h->g.aa || (h->g.tiled && (b.ex != h->g.ex || b.ey != h->g.ey || b.ez != h->g.ez)))
    return fail(LBM_EINVAL, "neighbouring slab has a different dtype, layout family, tile shape or x/y extent");
  const bool tile_aa = h->g.tiled && h->g.aa;
  if (b.pid == (int64_t)getpid()) {
    if (b.device != h->d.device) {
      int can = 0;
      CK(cudaDeviceCanAccessPeer(&can, h->d.device, b.device));
      if (!can) return fail(LBM_ENCCL, "device %d cannot access peer %d", h->d.device, b.device);
      cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return fail(LBM_ENCCL, "cudaDeviceEnablePeerAccess: %s", cudaGetErrorString(e));
      cudaGetLastError();
    }
    pr.f[0] = b.f[0];
    pr.f[1] = b.f[1];
    pr.sync = (unsigned long long*)b.sync;
    pr.rank = tile_aa ? (int*)b.rank : nullptr;
    pr.ipc = false;
  } else {
    CK(cudaIpcOpenMemHandle(&pr.f[0], b.ipc_f[0], cudaIpcMemLazyEnablePeerAccess));
    if (b.f[1] == b.f[0])  // A-A exporter: one buffer, mapped once
      pr.f[1] = pr.f[0];
    else
      CK(cudaIpcOpenMemHandle(&pr.f[1], b.ipc_f[1], cudaIpcMemLazyEnablePeerAccess));
    void* sy = nullptr;
    CK(cudaIpcOpenMemHandle(&sy, b.ipc_sync, cudaIpcMemLazyEnablePeerAccess));
    pr.sync = (unsigned long long*)sy;
    if (tile_aa) {
      void* rk = nullptr;
      CK(cudaIpcOpenMemHandle(&rk, b.ipc_rank, cudaIpcMemLazyEnablePeerAccess));
      pr.rank = (int*)rk;
    }
    pr.ipc = true;
  }
  pr.ps = b.ps;
  pr.nz = b.nz;
  pr.on = true;
  return 0;
}
}  // namespace

int lbm_halo_export(lbm_t* h, void* blob, size_t* bytes) {
  if (!h || !blob) return fail(LBM_EINVAL, "NULL argument");
  if (!h->geometry) return fail(LBM_ESTATE, "lbm_set_geometry must run before lbm_halo_export");
  if (h->g.tiled && !h->has_glo && !h->has_ghi)
    return fail(LBM_EINVAL, "this tile handle is not a z-slab (no ghost planes)");
  DeviceGuard dg(h->d.device);
  HaloBlob b;
  memset(&b, 0, sizeof(b));
  b.magic = kHaloMagic;
  b.device = h->d.device;
  b.esize = h->esize;
  b.nz = h->g.nz;
  b.ny = h->g.ny;
  b.nxp = h->g.nxp;
  b.pid = (int64_t)getpid();
  b.ps = h->g.ps;
  b.tiled = h->g.tiled;
  b.aa = h->g.aa;
  b.ex = h->g.ex;
  b.ey = h->g.ey;
  b.ez = h->g.ez;
  b.gz = h->g.gz;
  // dense: the PDF buffers (ghost planes inside); AB tiles: the ghost-plane
  // buffers; A-A tiles: the tile storage itself and its rank grid
  const bool tile_aa = h->g.tiled && h->g.aa;
  void* const* ex = (h->g.tiled && !tile_aa) ? h->gh : h->f;
  if (tile_aa) {
    b.rank = h->rank;
    CK(cudaIpcGetMemHandle(&b.ipc_rank, h->rank));
  }
  b.f[0] = ex[0];
  b.f[1] = ex[1] ? ex[1] : ex[0];  // A-A: one buffer
  b.sync = h->sync;
  CK(cudaIpcGetMemHandle(&b.ipc_f[0], b.f[0]));
  CK(cudaIpcGetMemHandle(&b.ipc_f[1], b.f[1]));
  CK(cudaIpcGetMemHandle(&b.ipc_sync, h->sync));
  memset(blob, 0, LBM_HALO_BLOB_BYTES);
  memcpy(blob, &b, sizeof(b));
  if (bytes) *bytes = LBM_HALO_BLOB_BYTES;
  return 0;
}

int lbm_halo_connect(lbm_t* h, const void* lo_blob, const void* hi_blob) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  if (!h->geometry) return fail(LBM_ESTATE, "lbm_set_geometry must run before lbm_halo_connect");
  if (h->g.tiled && !h->has_glo && !h->has_ghi && (lo_blob || hi_blob))
    return fail(LBM_EINVAL, "this tile handle is not a z-slab (no ghost planes)");
  if (h->g.pzw && (lo_blob || hi_blob))
    return fail(LBM_EINVAL, "a whole-domain periodic handle wraps z itself; it takes no halo");
  DeviceGuard dg(h->d.device);
  CK(cudaStreamSynchronize(h->stream));
  int rc = 0;
  HaloBlob b;
  if (lo_blob) {
    memcpy(&b, lo_blob, sizeof(b));
    if ((rc = open_peer(h, b, h->lo))) return rc;
  }
  if (hi_blob) {
    memcpy(&b, hi_blob, sizeof(b));
    if ((rc = open_peer(h, b, h->hi))) return rc;
  }
  if (h->esize == 4) preload_halo_kernels<float>(h); else preload_halo_kernels<double>(h);
  drop_graphs(h);  // captured step sequences change with the neighbours
  // capture and upload both parities' step graphs now, while no slab of this
  // process spins on a halo wait: instantiating them later, between launches
  // of neighbouring slabs driven from the same host thread, could wait behind
  // those spinning kernels
  if (h->use_graph && (h->lo.on || h->hi.on)) {
    if ((rc = capture_graph(h, 0)) || (rc = capture_graph(h, 1))) return rc;
    CK(cudaStreamSynchronize(h->stream));
  }
  h->halo_dirty = true;
  return 0;
}

}  // extern "C"

// ------------------------------------------------------- scalar host math
template <typename T>
static void to_t(const double* in, T* out, int n) {
  for (int k = 0; k < n; ++k) out[k] = (T)in[k];
}
template <typename T>
static void from_t(const T* in, double* out, int n) {
  for (int k = 0; k < n; ++k) out[k] = (double)in[k];
}

template <typename T>
static int feq_t(double rho, const double* u3, double* out) {
  T e[Q];
  feq19<T>((T)rho, (T)u3[0], (T)u3[1], (T)u3[2], e);
  from_t(e, out, Q);
  return 0;
}

extern "C" int lbm19_feq(int32_t dtype, double rho, const double* u3, double* out19) {
  if (!u3 || !out19) return fail(LBM_EINVAL, "NULL argument");
  return dtype == LBM_F32 ? feq_t<float>(rho, u3, out19) : feq_t<double>(rho, u3, out19);
}

template <typename T>
static int moments_t(const double* f19, double* rho, double* u3) {
  T f[Q], r, a, b, c;
  to_t(f19, f, Q);
  moments19<T>(f, r, a, b, c);
  *rho = r;
  u3[0] = a;
  u3[1] = b;
  u3[2] = c;
  return 0;
}

extern "C" int lbm19_moments(int32_t dtype, const double* f19, double* rho, double* u3) {
  if (!f19 || !rho || !u3) return fail(LBM_EINVAL, "NULL argument");
  return dtype == LBM_F32 ? moments_t<float>(f19, rho, u3) : moments_t<double>(f19, rho, u3);
}

template <typename T>
static int collide_t(const double* f19, double omega, double* out) {
  T f[Q], r, a, b, c;
  to_t(f19, f, Q);
  moments19<T>(f, r, a, b, c);
  collide19<T>(f, r, a, b, c, (T)omega);
  from_t(f, out, Q);
  return 0;
}

extern "C" int lbm19_collide(int32_t dtype, const double* f19, double omega, double* out19) {
  if (!f19 || !out19) return fail(LBM_EINVAL, "NULL argument");
  return dtype == LBM_F32 ? collide_t<float>(f19, omega, out19) : collide_t<double>(f19, omega, out19);
}

template <typename T>
static int zhv_t(const double* f19, int orient, const double* u3, double* out) {
  T f[Q];
  to_t(f19, f, Q);
  zou_he_velocity19<T>(f, (uint32_t)orient, (T)u3[0], (T)u3[1], (T)u3[2]);
  from_t(f, out, Q);
  return 0;
}

extern "C" int lbm19_zou_he_velocity(int32_t dtype, const double* f19, int32_t orient, const double* u3, double* out19) {
  if (!f19 || !u3 || !out19) return fail(LBM_EINVAL, "NULL argument");
  if (orient < O_NORTH || orient > O_BOTTOM) return fail(LBM_EINVAL, "orientation must name a face, got %d", orient);
  return dtype == LBM_F32 ? zhv_t<float>(f19, orient, u3, out19) : zhv_t<double>(f19, orient, u3, out19);
}

template <typename T>
static int zhp_t(const double* f19, int orient, double rw, double* out) {
  T f[Q];
  to_t(f19, f, Q);
  zou_he_pressure19<T>(f, (uint32_t)orient, (T)rw);
  from_t(f, out, Q);
  return 0;
}

extern "C" int lbm19_zou_he_pressure(int32_t dtype, const double* f19, int32_t orient, double rho_wall, double* out19) {
  if (!f19 || !out19) return fail(LBM_EINVAL, "NULL argument");
  if (orient < O_NORTH || orient > O_BOTTOM) return fail(LBM_EINVAL, "orientation must name a face, got %d", orient);
  return dtype == LBM_F32 ? zhp_t<float>(f19, orient, rho_wall, out19) : zhp_t<double>(f19, orient, rho_wall, out19);
}


