// sg_api.cu -- implementation of include/splinegpu.h (the C-ABI boundary).
//
// Built with nvcc for sm_100a into libsplinegpu.so.  The CUDA runtime is linked
// statically (no libcuda link-time dependency, so the library loads -- and its
// symbols can be checked -- on a machine without a GPU); NVRTC is linked
// dynamically from the image's CUDA 12.9 toolkit.  Generated kernels are loaded
// with the context-independent library API (cudaLibraryLoadData) and launched
// with cudaLaunchKernel, so no driver-API symbols are needed.
#include <cuda.h>  // CUtensorMap & friends (types only; the encoder is fetched at run time)
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/splinegpu.h"

#define SG_VERSION 100

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[2048];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(expr)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(SG_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,                 \
                  cudaGetErrorString(e_));                                             \
  } while (0)

size_t dtype_size(int dtype) { return dtype == SG_F64 ? 8 : 4; }

struct SgCosets {  // must match the struct emitted by cudagen.py
  const void* base[SG_MAX_COSETS];
};

struct SgTmaps {  // must match cudagen.py: one TMA descriptor per coset
  CUtensorMap m[SG_MAX_COSETS];
};

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  });
  return fn;
}

}  // namespace

struct sg_module {
  int device = 0;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kernel = nullptr;
  sg_module_info info{};
  // Launch slots: every launch gets its own 2-word slot of d_err -- [0] sticky error flags
  // (OR-ed over all slots by sg_module_status), [1] the tile / ray-block counter of the
  // persistent sorted and render kernels.  A slot is reused only after the launch that
  // last held it has finished (slot_ev), so launches of one module on different streams
  // never share a counter.
  static constexpr int kSlots = 16;
  unsigned* d_err = nullptr;
  cudaEvent_t slot_ev[kSlots] = {};
  unsigned slot_next = 0;
  std::mutex slot_mu;
  int regs = 0, local_bytes = 0;
  std::mutex mu;  // guards the host-path scratch below
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  cudaStream_t streams[3] = {nullptr, nullptr, nullptr};
  // binned mode: sorted queries + per-bin counts/starts/cursors (one stream at a time)
  std::mutex bin_mu;
  // the binning scratch is one buffer per module: launches on different streams (the
  // pipelined host path, or callers) are ordered behind the previous one with this event
  cudaEvent_t bin_done = nullptr;
  void* bin_scratch = nullptr;
  size_t bin_scratch_bytes = 0;
  int64_t nbins = 0;
  int64_t nb[SG_MAX_DIM] = {1, 1, 1, 1};
  // optional event timing of the evaluation kernel
  bool timing = false;
  std::mutex t_mu;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> t_events;
  size_t t_used = 0;
};

// Optional L2 residency control (env SPLINEGPU_L2_PERSIST=1): launches carry an access
// policy window over the coefficient volume (persisting hits, streaming misses) so the
// query/result streams cannot evict it.  Returns the persisting budget (0 = disabled).
static size_t l2_persist_budget(int device) {
  static std::mutex mu;
  static int state[64] = {};      // 0 unknown, 1 off, 2 on
  static size_t budget[64] = {};
  static size_t max_window[64] = {};
  std::lock_guard<std::mutex> lock(mu);
  if (device < 0 || device >= 64) return 0;
  if (state[device] == 0) {
    state[device] = 1;
    const char* e = getenv("SPLINEGPU_L2_PERSIST");
    if (e && atoi(e) > 0) {
      int mx = 0, win = 0;
      cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, device);
      cudaDeviceGetAttribute(&win, cudaDevAttrMaxAccessPolicyWindowSize, device);
      if (mx > 0 && win > 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)mx) == cudaSuccess) {
        budget[device] = (size_t)mx;
        max_window[device] = (size_t)win;
        state[device] = 2;
      }
      cudaGetLastError();
    }
  }
  return state[device] == 2 ? std::min(budget[device], max_window[device]) : 0;
}

// Take the next launch slot for a launch on `st` (see sg_module::d_err): the stream waits
// for the slot's previous holder, the slot's counter is zeroed when the kernel uses one.
// The caller keeps `lk` until it has recorded the slot event (release_slot) after the
// launch, so no other launch can take the same slot in between.
static int acquire_slot(sg_module* m, cudaStream_t st, bool zero_counter,
                        std::unique_lock<std::mutex>& lk, int* slot, unsigned** err) {
  lk = std::unique_lock<std::mutex>(m->slot_mu);
  const int k = (int)(m->slot_next++ % sg_module::kSlots);
  if (!m->slot_ev[k]) CU(cudaEventCreateWithFlags(&m->slot_ev[k], cudaEventDisableTiming));
  else CU(cudaStreamWaitEvent(st, m->slot_ev[k], 0));
  if (zero_counter) CU(cudaMemsetAsync(m->d_err + 2 * k + 1, 0, sizeof(unsigned), st));
  *slot = k;
  *err = m->d_err + 2 * k;
  return SG_OK;
}

static int release_slot(sg_module* m, int k, cudaStream_t st) {
  CU(cudaEventRecord(m->slot_ev[k], st));
  return SG_OK;
}

static int timed_launch(sg_module* m, const void* func, dim3 grid, dim3 block, void** args,
                        size_t smem, cudaStream_t st, const void* win_base = nullptr,
                        size_t win_bytes = 0) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (m->timing) {
    std::lock_guard<std::mutex> lock(m->t_mu);
    if (m->t_used == m->t_events.size()) {
      cudaEvent_t a, b;
      CU(cudaEventCreate(&a));
      CU(cudaEventCreate(&b));
      m->t_events.emplace_back(a, b);
    }
    e0 = m->t_events[m->t_used].first;
    e1 = m->t_events[m->t_used].second;
    ++m->t_used;
    CU(cudaEventRecord(e0, st));
  }
  const size_t budget = win_base ? l2_persist_budget(m->device) : 0;
  if (budget) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeAccessPolicyWindow;
    const size_t nb = std::min(win_bytes, budget);
    at[0].val.accessPolicyWindow.base_ptr = const_cast<void*>(win_base);
    at[0].val.accessPolicyWindow.num_bytes = nb;
    at[0].val.accessPolicyWindow.hitRatio = std::min(1.0f, (float)budget / (float)std::max<size_t>(nb, 1));
    at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CU(cudaLaunchKernelExC(&cfg, func, args));
  } else {
    CU(cudaLaunchKernel(func, grid, block, args, smem, st));
  }
  if (e1) CU(cudaEventRecord(e1, st));
  return SG_OK;
}

struct sg_volume {
  int device = 0;
  int dim = 0, ncosets = 0, halo = 0, dtype = SG_F32;
  int64_t ext[SG_MAX_COSETS][SG_MAX_DIM] = {};
  int64_t pext[SG_MAX_COSETS][SG_MAX_DIM] = {};
  void* alloc = nullptr;  // one allocation, coset-split
  size_t bytes = 0;
  size_t coset_off[SG_MAX_COSETS] = {};  // byte offset of each coset's padded array
  const void* origin[SG_MAX_COSETS] = {};  // padded element (h, h, ..., h)
  // linear-fetch modules (SG_MODE_LINEAR): one filtered, wrapping f32 texture per coset,
  // built from the volume on first use (volume_textures) and owned by the volume
  cudaArray_t tarr[SG_MAX_COSETS] = {};
  unsigned long long tex[SG_MAX_COSETS] = {};
  bool tex_ready = false;
};

struct SgTex {  // must match linfetch.py
  unsigned long long t[SG_MAX_COSETS];
};

static std::mutex g_tex_mu;

static void volume_textures_free(sg_volume* v) {
  for (int c = 0; c < SG_MAX_COSETS; ++c) {
    if (v->tex[c]) cudaDestroyTextureObject((cudaTextureObject_t)v->tex[c]);
    if (v->tarr[c]) cudaFreeArray(v->tarr[c]);
    v->tex[c] = 0;
    v->tarr[c] = nullptr;
  }
  v->tex_ready = false;
}

// Texture objects of a volume (built once): the unpadded coset arrays are copied from the
// padded allocation into cudaArrays (axis s-1 -> texture x), sampled with normalized
// coordinates, wrap addressing (the reference's periodic fetch) and linear filtering.
static int volume_textures(sg_volume* v, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(g_tex_mu);
  if (v->tex_ready) return SG_OK;
  if (v->dtype != SG_F32 || v->dim > 3)
    return fail(SG_EINVAL, "linear fetch needs an f32 volume of dimension <= 3");
  for (int c = 0; c < v->ncosets; ++c) {
    const int s = v->dim;
    const size_t w = (size_t)v->ext[c][s - 1];
    const size_t h = s >= 2 ? (size_t)v->ext[c][s - 2] : 0;
    const size_t d = s >= 3 ? (size_t)v->ext[c][s - 3] : 0;
    cudaChannelFormatDesc desc = cudaCreateChannelDesc<float>();
    cudaError_t e = cudaMalloc3DArray(&v->tarr[c], &desc, make_cudaExtent(w, h, d));
    if (e != cudaSuccess) {
      volume_textures_free(v);
      return fail(SG_ENOMEM, "cudaMalloc3DArray: %s", cudaGetErrorString(e));
    }
    cudaMemcpy3DParms p{};
    const size_t pw = (size_t)v->pext[c][s - 1];
    const size_t ph = s >= 2 ? (size_t)v->pext[c][s - 2] : 1;
    p.srcPtr = make_cudaPitchedPtr(const_cast<void*>(v->origin[c]), pw * sizeof(float), w, ph);
    p.dstArray = v->tarr[c];
    p.extent = make_cudaExtent(w, h ? h : 1, d ? d : 1);
    p.kind = cudaMemcpyDeviceToDevice;
    e = cudaMemcpy3DAsync(&p, st);
    if (e == cudaSuccess) {
      cudaResourceDesc rd{};
      rd.resType = cudaResourceTypeArray;
      rd.res.array.array = v->tarr[c];
      cudaTextureDesc td{};
      for (int a = 0; a < 3; ++a) td.addressMode[a] = cudaAddressModeWrap;
      td.filterMode = cudaFilterModeLinear;
      td.readMode = cudaReadModeElementType;
      td.normalizedCoords = 1;
      cudaTextureObject_t t = 0;
      e = cudaCreateTextureObject(&t, &rd, &td, nullptr);
      v->tex[c] = (unsigned long long)t;
    }
    if (e != cudaSuccess) {
      volume_textures_free(v);
      return fail(SG_ECUDA, "volume texture: %s", cudaGetErrorString(e));
    }
  }
  v->tex_ready = true;
  return SG_OK;
}

// Periodic ghost-halo fill: dst (padded, C order) <- src (unpadded, C order).
template <typename T>
__global__ void sg_pad_kernel(T* __restrict__ dst, const T* __restrict__ src, int dim,
                              long long p0, long long p1, long long p2, long long p3,
                              long long e0, long long e1, long long e2, long long e3, int h,
                              long long total) {
  long long pe[4] = {p0, p1, p2, p3};
  long long ee[4] = {e0, e1, e2, e3};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    long long rem = i, src_idx = 0, mul = 1;
    long long coord[4];
    for (int d = dim - 1; d >= 0; --d) {
      coord[d] = rem % pe[d];
      rem /= pe[d];
    }
    for (int d = dim - 1; d >= 0; --d) {
      long long c = coord[d] - h;
      c %= ee[d];
      if (c < 0) c += ee[d];
      src_idx += c * mul;
      mul *= ee[d];
    }
    dst[i] = src[src_idx];
  }
}


// ---- binned mode: counting sort of the queries by cell ---------------------------------
//
// Bins partition the periodic box of coset 0 into cubes of `bin` cells.  The bin of a
// query is computed in cheap f32 arithmetic from the wrapped coordinate; the generated
// kernel recomputes the exact fp64 lattice shift and tolerates a one-cell disagreement
// at bin borders (its brick carries a margin of reach + 2 cells, and the brick-local
// index is wrapped modulo the extent), so bins only need to be *approximately* right.
struct BinGeom {
  int dim, bin;
  float ext[3];
  float inv_ext[3];
  float inv_bin;
  int nb[3];
  long long nbins;
};


constexpr int SG_SORT_THREADS = 1024;
constexpr int SG_SMEM_BINS = 16384;     // bins that fit the privatized shared histograms

__device__ __forceinline__ int sg_bin_xyz(float x, float y, float z, const BinGeom& g) {
  const float c[3] = {x, y, z};
  int lin = 0;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if (d < g.dim) {
      float xw = c[d] - g.ext[d] * floorf(c[d] * g.inv_ext[d]);
      int b = (int)floorf(xw * g.inv_bin);
      b = min(max(b, 0), g.nb[d] - 1);
      lin = lin * g.nb[d] + b;
    }
  }
  return lin;
}


// Queries of a CTA range are read as float4 triples (4 queries of 3 floats) when the
// range is 16-B aligned; `visit(i, x, y, z)` is called for every query.
template <typename F>
__device__ __forceinline__ void sg_for_queries(const float* __restrict__ xs, long long lo,
                                               long long hi, const BinGeom& g, F visit) {
  if (g.dim == 3 && ((lo & 3) == 0) && ((((uintptr_t)xs) & 15) == 0)) {
    const float4* X4 = reinterpret_cast<const float4*>(xs);
    const long long g0 = lo >> 2, g1 = hi >> 2;   // full groups
    for (long long q = g0 + threadIdx.x; q < g1; q += blockDim.x) {
      const float4 a = X4[3 * q], b = X4[3 * q + 1], c = X4[3 * q + 2];
      const long long i = q << 2;
      visit(i, a.x, a.y, a.z);
      visit(i + 1, a.w, b.x, b.y);
      visit(i + 2, b.z, b.w, c.x);
      visit(i + 3, c.y, c.z, c.w);
    }
    for (long long i = (g1 << 2) + threadIdx.x; i < hi; i += blockDim.x)
      visit(i, xs[i * 3], xs[i * 3 + 1], xs[i * 3 + 2]);
  } else {
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x)
      visit(i, xs[i * g.dim], g.dim > 1 ? xs[i * g.dim + 1] : 0.f,
            g.dim > 2 ? xs[i * g.dim + 2] : 0.f);
  }
}

// K1: per-CTA histogram of a contiguous query range -> mat[bin * G + cta] (smem atomics),
// and the per-bin totals (one global atomic per non-empty (CTA, bin)).
__global__ void __launch_bounds__(SG_SORT_THREADS) sg_bin_count(
    const float* __restrict__ xs, long long n, long long per, BinGeom g,
    int* __restrict__ mat, int* __restrict__ bin_tot) {
  extern __shared__ int hist[];
  const int G = gridDim.x;
  for (int b = threadIdx.x; b < g.nbins; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const long long lo = (long long)blockIdx.x * per;
  const long long hi = min(n, lo + per);
  sg_for_queries(xs, lo, hi, g, [&](long long, float x, float y, float z) {
    atomicAdd(&hist[sg_bin_xyz(x, y, z, g)], 1);
  });
  __syncthreads();
  for (int b = threadIdx.x; b < g.nbins; b += blockDim.x) {
    const int h = hist[b];
    mat[(long long)b * G + blockIdx.x] = h;
    if (h) atomicAdd(&bin_tot[b], h);
  }
}

// block-wide exclusive scan (any multiple-of-32 block size up to 1024)
__device__ __forceinline__ int sg_block_excl_scan(int v, int* sh, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    sh[lane] = t;
  }
  __syncthreads();
  int excl = x - v + (w ? sh[w - 1] : 0);
  if (total) *total = sh[(blockDim.x >> 5) - 1];
  __syncthreads();
  return excl;
}





// One CTA: bin starts (exclusive scan of the bin totals), the scatter cursors, the
// evaluation work items; re-zeroes the totals for the next call.  Each scatter CTA then
// reserves its (bin) ranges with one atomicAdd on the cursor per bin, so no scan of the
// (bin x CTA) count matrix is needed.
__global__ void __launch_bounds__(1024) sg_bin_plan(int* __restrict__ bin_tot, int nbins, long long n,
                                                    int chunk, int* __restrict__ starts,
                                                    int* __restrict__ cursor,
                                                    int2* __restrict__ items, int max_items) {
  __shared__ int sh[32];
  const int per = (nbins + 1023) / 1024;
  const int lo = threadIdx.x * per, hi = min(nbins, lo + per);
  int mine = 0;
  for (int b = lo; b < hi; ++b) mine += bin_tot[b];
  int at = sg_block_excl_scan(mine, sh, nullptr);
  int nchunks = 0;
  for (int b = lo; b < hi; ++b) {
    const int t = bin_tot[b];
    starts[b] = at;
    cursor[b] = at;
    bin_tot[b] = 0;
    nchunks += (t + chunk - 1) / chunk;
    at += t;
  }
  if (threadIdx.x == 1023) starts[nbins] = (int)n;
  int total;
  int it = sg_block_excl_scan(nchunks, sh, &total);
  __syncthreads();
  for (int b = lo; b < hi; ++b) {
    const int s0 = starts[b], s1 = starts[b + 1];
    for (int q = s0; q < s1; q += chunk) items[it++] = make_int2(b, q);
  }
  for (int i = total + threadIdx.x; i < max_items; i += 1024) items[i] = make_int2(-1, 0);
}

// K3: scatter (x, y, z, index) records to their sorted positions
__global__ void __launch_bounds__(SG_SORT_THREADS) sg_bin_scatter(
    const float* __restrict__ xs, long long n, long long per, BinGeom g,
    const int* __restrict__ mat, int* __restrict__ cursor, float4* __restrict__ sorted) {
  extern __shared__ int sh[];
  int* cnt = sh;   // running position per bin: this CTA's reserved range in each bin
  const int G = gridDim.x;
  for (int b = threadIdx.x; b < g.nbins; b += blockDim.x) {
    const int c = mat[(long long)b * G + blockIdx.x];
    cnt[b] = c ? atomicAdd(&cursor[b], c) : 0;
  }
  __syncthreads();
  const long long lo = (long long)blockIdx.x * per;
  const long long hi = min(n, lo + per);
  sg_for_queries(xs, lo, hi, g, [&](long long i, float x, float y, float z) {
    const int pos = atomicAdd(&cnt[sg_bin_xyz(x, y, z, g)], 1);
    sorted[pos] = make_float4(x, y, z, __int_as_float((int)i));
  });
}


// K3': tile-local counting sort before the scatter: records of one bin leave the CTA as
// contiguous runs (coalesced 16-B stores) instead of one scattered store per query.
constexpr int SG_TILED_MAX_BINS_CAP = 10240;   // smem: 4 ints per bin + the tile's records
// per-tile histogram cost grows with the bin count: the tiled scatter is used up to this many
// bins (env SPLINEGPU_TILED_MAX_BINS, at most SG_TILED_MAX_BINS_CAP), the plain one above
static int sg_tiled_max_bins() {
  static const int v = [] {
    const char* e = getenv("SPLINEGPU_TILED_MAX_BINS");
    const int x = e ? atoi(e) : 2048;
    return x >= 0 && x <= SG_TILED_MAX_BINS_CAP ? x : 2048;
  }();
  return v;
}

template <int THREADS, int GROUPS>
__global__ void __launch_bounds__(THREADS) sg_bin_scatter_tiled(
    const float* __restrict__ xs, long long n, long long per, BinGeom g,
    const int* __restrict__ mat, int* __restrict__ cursor, float4* __restrict__ sorted) {
  constexpr int TILE = 4 * THREADS * GROUPS;   // records per tile: GROUPS x 4 per thread
  extern __shared__ __align__(16) unsigned char shb[];
  const int nb = (int)g.nbins;
  float4* tile = reinterpret_cast<float4*>(shb);                 // TILE records
  int* tdst = reinterpret_cast<int*>(tile + TILE);                // TILE destinations
  int* gpos = tdst + TILE;                                         // nb: global cursor
  int* lcnt = gpos + nb;                                           // nb: tile counts
  int* loff = lcnt + nb;                                           // nb: tile offsets
  int* gbase = loff + nb;                                          // nb: this tile's global base
  __shared__ int scan_sh[32];
  const int G = gridDim.x;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const int c = mat[(long long)b * G + blockIdx.x];
    gpos[b] = c ? atomicAdd(&cursor[b], c) : 0;
    lcnt[b] = 0;
  }
  __syncthreads();
  const long long lo = (long long)blockIdx.x * per;
  const long long hi = min(n, lo + per);
  const bool vec = g.dim == 3 && ((((uintptr_t)xs) & 15) == 0);
  // software pipeline: the next tile's query triples are loaded while this tile is sorted
  float4 pa[GROUPS], pb[GROUPS], pc[GROUPS];
#pragma unroll
  for (int gi = 0; gi < GROUPS; ++gi) {
    pa[gi] = pb[gi] = pc[gi] = make_float4(0.f, 0.f, 0.f, 0.f);
    const long long q = lo + gi * 4 * THREADS + threadIdx.x * 4;
    if (vec && q + 4 <= hi) {
      const float4* X4 = reinterpret_cast<const float4*>(xs + q * 3);
      pa[gi] = X4[0];
      pb[gi] = X4[1];
      pc[gi] = X4[2];
    }
  }
  for (long long t0 = lo; t0 < hi; t0 += TILE) {
    const int tn = (int)min((long long)TILE, hi - t0);
    float4 rec[4 * GROUPS];
    int bb[4 * GROUPS], rk[4 * GROUPS];
#pragma unroll
    for (int gi = 0; gi < GROUPS; ++gi) {
      const int q0 = gi * 4 * THREADS + threadIdx.x * 4;
      const float4 ca = pa[gi], cb = pb[gi], cc = pc[gi];
      {
        const long long nx = t0 + TILE + q0;
        if (vec && nx + 4 <= hi) {
          const float4* X4 = reinterpret_cast<const float4*>(xs + nx * 3);
          pa[gi] = __ldg(X4);
          pb[gi] = __ldg(X4 + 1);
          pc[gi] = __ldg(X4 + 2);
        }
      }
      // A: 4 consecutive queries per thread and group (one float4 triple when aligned)
#pragma unroll
      for (int k = 0; k < 4; ++k) bb[4 * gi + k] = -1;
      if (q0 < tn) {
        const long long i0 = t0 + q0;
        if (vec && q0 + 4 <= tn) {
          rec[4 * gi + 0] = make_float4(ca.x, ca.y, ca.z, __int_as_float((int)i0));
          rec[4 * gi + 1] = make_float4(ca.w, cb.x, cb.y, __int_as_float((int)(i0 + 1)));
          rec[4 * gi + 2] = make_float4(cb.z, cb.w, cc.x, __int_as_float((int)(i0 + 2)));
          rec[4 * gi + 3] = make_float4(cc.y, cc.z, cc.w, __int_as_float((int)(i0 + 3)));
#pragma unroll
          for (int k = 0; k < 4; ++k)
            bb[4 * gi + k] = sg_bin_xyz(rec[4 * gi + k].x, rec[4 * gi + k].y, rec[4 * gi + k].z, g);
        } else {
          for (int k = 0; k < 4 && q0 + k < tn; ++k) {
            const long long i = i0 + k;
            rec[4 * gi + k] = make_float4(xs[i * g.dim], g.dim > 1 ? xs[i * g.dim + 1] : 0.f,
                                          g.dim > 2 ? xs[i * g.dim + 2] : 0.f, __int_as_float((int)i));
            bb[4 * gi + k] = sg_bin_xyz(rec[4 * gi + k].x, rec[4 * gi + k].y, rec[4 * gi + k].z, g);
          }
        }
      }
    }
    // (lcnt is zero here: cleared at start, then by phase B of the previous tile)
#pragma unroll
    for (int k = 0; k < 4 * GROUPS; ++k)
      if (bb[k] >= 0) rk[k] = atomicAdd(&lcnt[bb[k]], 1);
    __syncthreads();
    // B: tile offsets (exclusive scan over bins), this tile's global bases, counts reset
    {
      const int per_t = (nb + THREADS - 1) / THREADS;
      const int b0 = threadIdx.x * per_t, b1 = min(nb, b0 + per_t);
      int mine = 0;
      for (int b = b0; b < b1; ++b) mine += lcnt[b];
      int at = sg_block_excl_scan(mine, scan_sh, nullptr);
      for (int b = b0; b < b1; ++b) {
        const int c = lcnt[b];
        loff[b] = at;
        gbase[b] = gpos[b];   // this tile's records of bin b start here in the output
        gpos[b] += c;
        lcnt[b] = 0;          // ready for the next tile's phase A
        at += c;
      }
    }
    __syncthreads();
    // C: place records bin-contiguously in the tile, each with its final destination
#pragma unroll
    for (int k = 0; k < 4 * GROUPS; ++k)
      if (bb[k] >= 0) {
        const int slot = loff[bb[k]] + rk[k];
        tile[slot] = rec[k];
        tdst[slot] = gbase[bb[k]] + rk[k];
      }
    __syncthreads();
    // D: coalesced runs to the global positions
    for (int j = threadIdx.x; j < tn; j += blockDim.x) sorted[tdst[j]] = tile[j];
    __syncthreads();
  }
}

extern "C" {

int sg_version(void) { return SG_VERSION; }

const char* sg_last_error(void) { return g_err.c_str(); }

int sg_device_count(int* count) {
  if (!count) return fail(SG_EINVAL, "count is NULL");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    cudaGetLastError();
    return fail(SG_ECUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  *count = n;
  return SG_OK;
}

void sg_free(void* p) { free(p); }

int sg_compile(const char* source, const char* name, const char* const* opts, int nopts,
               void** image, size_t* image_len, char** log) {
  if (!source || !image || !image_len) return fail(SG_EINVAL, "NULL argument");
  nvrtcProgram prog;
  nvrtcResult r = nvrtcCreateProgram(&prog, source, name ? name : "sg_kernel.cu", 0,
                                     nullptr, nullptr);
  if (r != NVRTC_SUCCESS) return fail(SG_ECOMPILE, "nvrtcCreateProgram: %s", nvrtcGetErrorString(r));
  std::vector<const char*> o;
  bool has_arch = false;
  for (int i = 0; i < nopts; ++i) {
    o.push_back(opts[i]);
    if (strstr(opts[i], "arch") != nullptr) has_arch = true;
  }
  if (!has_arch) o.push_back("--gpu-architecture=sm_100a");
  r = nvrtcCompileProgram(prog, (int)o.size(), o.data());
  size_t log_len = 0;
  nvrtcGetProgramLogSize(prog, &log_len);
  std::string lg(log_len, '\0');
  if (log_len) nvrtcGetProgramLog(prog, &lg[0]);
  if (log) {
    *log = (char*)malloc(lg.size() + 1);
    memcpy(*log, lg.c_str(), lg.size() + 1);
  }
  if (r != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return fail(SG_ECOMPILE, "nvrtc: %s\n%s", nvrtcGetErrorString(r), lg.c_str());
  }
  size_t n = 0;
  r = nvrtcGetCUBINSize(prog, &n);
  if (r != NVRTC_SUCCESS || n == 0) {
    nvrtcDestroyProgram(&prog);
    return fail(SG_ECOMPILE, "nvrtcGetCUBINSize: %s (did the options name an sm_ arch?)",
                nvrtcGetErrorString(r));
  }
  void* buf = malloc(n);
  r = nvrtcGetCUBIN(prog, (char*)buf);
  nvrtcDestroyProgram(&prog);
  if (r != NVRTC_SUCCESS) {
    free(buf);
    return fail(SG_ECOMPILE, "nvrtcGetCUBIN: %s", nvrtcGetErrorString(r));
  }
  *image = buf;
  *image_len = n;
  return SG_OK;
}

int sg_module_load(const void* image, size_t image_len, const char* entry, int device,
                   const sg_module_info* info, sg_module** out) {
  if (!image || !entry || !info || !out) return fail(SG_EINVAL, "NULL argument");
  if (image_len < 16) return fail(SG_EINVAL, "image of %zu bytes is not a cubin", image_len);
  if (info->dim < 1 || info->dim > SG_MAX_DIM) return fail(SG_EINVAL, "bad dim %d", info->dim);
  if (info->ncosets < 1 || info->ncosets > SG_MAX_COSETS)
    return fail(SG_EINVAL, "bad coset count %d", info->ncosets);
  if (info->block < 32 || info->block > 1024) return fail(SG_EINVAL, "bad block %d", info->block);
  CU(cudaSetDevice(device));
  sg_module* m = new sg_module();
  m->device = device;
  m->info = *info;
  if (m->info.queries_per_thread < 1) m->info.queries_per_thread = 1;
  cudaError_t e = cudaLibraryLoadData(&m->lib, image, nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e != cudaSuccess) {
    delete m;
    return fail(SG_ECUDA, "cudaLibraryLoadData: %s", cudaGetErrorString(e));
  }
  e = cudaLibraryGetKernel(&m->kernel, m->lib, entry);
  if (e != cudaSuccess) {
    cudaLibraryUnload(m->lib);
    delete m;
    return fail(SG_ECUDA, "cudaLibraryGetKernel(%s): %s", entry, cudaGetErrorString(e));
  }
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, (const void*)m->kernel) == cudaSuccess) {
    m->regs = fa.numRegs;
    m->local_bytes = (int)fa.localSizeBytes;
  } else {
    cudaGetLastError();
  }
  if (m->info.mode == SG_MODE_BINNED) {
    if (m->info.dtype != SG_F32 || m->info.dim > 3) {
      cudaLibraryUnload(m->lib);
      delete m;
      return fail(SG_EINVAL, "binned mode supports f32 volumes of dimension <= 3");
    }
    m->nbins = 1;
    for (int d = 0; d < m->info.dim; ++d) {
      m->nb[d] = (m->info.extents[d] + m->info.bin - 1) / m->info.bin;
      m->nbins *= m->nb[d];
    }
    if (m->nbins > (1LL << 30)) {
      cudaLibraryUnload(m->lib);
      delete m;
      return fail(SG_EINVAL, "too many bins");
    }
    {
      e = cudaFuncSetAttribute((const void*)m->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               m->info.smem_bytes);
      if (e != cudaSuccess) {
        cudaLibraryUnload(m->lib);
        delete m;
        cudaGetLastError();   // clear the non-sticky error so later calls do not report it
        return fail(SG_ECUDA, "smem attribute: %s", cudaGetErrorString(e));
      }
    }
  }
  if (m->info.mode == SG_MODE_LINEAR && (m->info.dtype != SG_F32 || m->info.dim > 3)) {
    cudaLibraryUnload(m->lib);
    delete m;
    return fail(SG_EINVAL, "linear-fetch modules filter f32 volumes of dimension <= 3");
  }
  if (m->info.mode == SG_MODE_DIRECT && m->info.presort) {
    if (m->info.dtype != SG_F32 || m->info.dim > 3 || m->info.bin < 1) {
      cudaLibraryUnload(m->lib);
      delete m;
      return fail(SG_EINVAL, "presort needs f32 queries of dimension <= 3 and a bin >= 1");
    }
    m->nbins = 1;
    for (int d = 0; d < m->info.dim; ++d) {
      m->nb[d] = (m->info.extents[d] + m->info.bin - 1) / m->info.bin;
      m->nbins *= m->nb[d];
    }
  }
  if ((m->info.mode == SG_MODE_DIRECT || m->info.mode == SG_MODE_RENDER) && m->info.smem_bytes > 0) {
    // sorted direct kernels keep their per-tile pair records in dynamic shared memory
    e = cudaFuncSetAttribute((const void*)m->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             m->info.smem_bytes);
    if (e != cudaSuccess) {
      cudaLibraryUnload(m->lib);
      delete m;
      cudaGetLastError();
      return fail(SG_ECUDA, "smem attribute: %s", cudaGetErrorString(e));
    }
  }
  // launch slots: [2k] sticky error flags, [2k + 1] tile counter (zeroed per launch)
  e = cudaMalloc(&m->d_err, 2 * sg_module::kSlots * sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemset(m->d_err, 0, 2 * sg_module::kSlots * sizeof(unsigned));
  if (e != cudaSuccess) {
    cudaLibraryUnload(m->lib);
    delete m;
    return fail(SG_ECUDA, "error-word alloc: %s", cudaGetErrorString(e));
  }
  *out = m;
  return SG_OK;
}

int sg_module_free(sg_module* m) {
  if (!m) return SG_OK;
  cudaSetDevice(m->device);
  for (auto& s : m->streams)
    if (s) cudaStreamDestroy(s);
  if (m->scratch) cudaFree(m->scratch);
  if (m->bin_scratch) cudaFree(m->bin_scratch);
  if (m->bin_done) cudaEventDestroy(m->bin_done);
  for (auto& ev : m->slot_ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& pr : m->t_events) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  if (m->d_err) cudaFree(m->d_err);
  if (m->lib) cudaLibraryUnload(m->lib);
  delete m;
  return SG_OK;
}

int sg_module_timing(sg_module* m, int enable) {
  if (!m) return fail(SG_EINVAL, "NULL module");
  m->timing = enable != 0;
  return SG_OK;
}

int sg_module_kernel_time(sg_module* m, double* total_ms, int64_t* launches) {
  if (!m) return fail(SG_EINVAL, "NULL module");
  std::lock_guard<std::mutex> lock(m->t_mu);
  double tot = 0;
  for (size_t i = 0; i < m->t_used; ++i) {
    CU(cudaEventSynchronize(m->t_events[i].second));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, m->t_events[i].first, m->t_events[i].second));
    tot += ms;
  }
  if (total_ms) *total_ms = tot;
  if (launches) *launches = (int64_t)m->t_used;
  m->t_used = 0;
  return SG_OK;
}

int sg_module_regs(const sg_module* m, int* regs, int* local_bytes) {
  if (!m) return fail(SG_EINVAL, "NULL module");
  if (regs) *regs = m->regs;
  if (local_bytes) *local_bytes = m->local_bytes;
  return SG_OK;
}

int sg_module_status(sg_module* m, void* stream, uint32_t* flags) {
  if (!m) return fail(SG_EINVAL, "NULL module");
  CU(cudaSetDevice(m->device));
  unsigned w[2 * sg_module::kSlots] = {};
  cudaStream_t st = (cudaStream_t)stream;
  CU(cudaMemcpyAsync(w, m->d_err, sizeof w, cudaMemcpyDeviceToHost, st));
  // clear the error words only: a counter may belong to a launch running on another stream
  CU(cudaMemset2DAsync(m->d_err, 2 * sizeof(unsigned), 0, sizeof(unsigned), sg_module::kSlots, st));
  CU(cudaStreamSynchronize(st));
  unsigned h = 0;
  for (int k = 0; k < sg_module::kSlots; ++k) h |= w[2 * k];
  if (flags) *flags = h;
  if (h & 1u) return fail(SG_EUNREACHABLE, "point classified into an unreachable sigma entry");
  return SG_OK;
}

int sg_volume_create(int device, int dim, int ncosets, const int64_t* extents, int halo,
                     const int64_t* padded, int dtype, const void* const* src,
                     int src_on_device, void* stream, sg_volume** out) {
  if (!extents || !src || !out) return fail(SG_EINVAL, "NULL argument");
  if (dim < 1 || dim > SG_MAX_DIM) return fail(SG_EINVAL, "bad dim %d", dim);
  if (ncosets < 1 || ncosets > SG_MAX_COSETS) return fail(SG_EINVAL, "bad coset count %d", ncosets);
  if (halo < 0) return fail(SG_EINVAL, "negative halo");
  if (dtype != SG_F32 && dtype != SG_F64) return fail(SG_EINVAL, "bad dtype %d", dtype);
  CU(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  sg_volume* v = new sg_volume();
  v->device = device;
  v->dim = dim;
  v->ncosets = ncosets;
  v->halo = halo;
  v->dtype = dtype;
  const size_t es = dtype_size(dtype);
  size_t off = 0;
  for (int c = 0; c < ncosets; ++c) {
    int64_t n = 1;
    for (int d = 0; d < dim; ++d) {
      int64_t e = extents[c * dim + d];
      if (e < 1) {
        delete v;
        return fail(SG_EINVAL, "extents must be positive");
      }
      v->ext[c][d] = e;
      v->pext[c][d] = padded ? padded[c * dim + d] : e + 2 * halo;
      if (v->pext[c][d] < e + halo) {
        delete v;
        return fail(SG_EINVAL, "padded extent %lld too small for extent %lld + halo %d",
                    (long long)v->pext[c][d], (long long)e, halo);
      }
      n *= v->pext[c][d];
    }
    off = (off + 255) & ~size_t(255);
    v->coset_off[c] = off;
    off += (size_t)n * es;
  }
  v->bytes = off;
  cudaError_t e = cudaMalloc(&v->alloc, v->bytes);
  if (e != cudaSuccess) {
    delete v;
    return fail(SG_ENOMEM, "cudaMalloc(%zu): %s", off, cudaGetErrorString(e));
  }
  for (int c = 0; c < ncosets; ++c) {
    int64_t n = 1, np = 1;
    for (int d = 0; d < dim; ++d) {
      n *= v->ext[c][d];
      np *= v->pext[c][d];
    }
    const void* s = src[c];
    void* tmp = nullptr;
    if (!src_on_device) {
      e = cudaMalloc(&tmp, (size_t)n * es);
      if (e == cudaSuccess) e = cudaMemcpyAsync(tmp, s, (size_t)n * es, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) {
        if (tmp) cudaFree(tmp);
        cudaFree(v->alloc);
        delete v;
        return fail(SG_ECUDA, "volume upload: %s", cudaGetErrorString(e));
      }
      s = tmp;
    }
    long long pe[4] = {1, 1, 1, 1}, ee[4] = {1, 1, 1, 1};
    for (int d = 0; d < dim; ++d) {
      pe[d] = v->pext[c][d];
      ee[d] = v->ext[c][d];
    }
    char* dst = (char*)v->alloc + v->coset_off[c];
    int blocks = (int)std::min<long long>((np + 255) / 256, 148LL * 16);
    if (dtype == SG_F32)
      sg_pad_kernel<float><<<blocks, 256, 0, st>>>((float*)dst, (const float*)s, dim, pe[0],
                                                   pe[1], pe[2], pe[3], ee[0], ee[1], ee[2],
                                                   ee[3], halo, np);
    else
      sg_pad_kernel<double><<<blocks, 256, 0, st>>>((double*)dst, (const double*)s, dim, pe[0],
                                                    pe[1], pe[2], pe[3], ee[0], ee[1], ee[2],
                                                    ee[3], halo, np);
    e = cudaGetLastError();
    if (e == cudaSuccess && tmp) e = cudaStreamSynchronize(st);
    if (tmp) cudaFree(tmp);
    if (e != cudaSuccess) {
      cudaFree(v->alloc);
      delete v;
      return fail(SG_ECUDA, "halo fill: %s", cudaGetErrorString(e));
    }
    // origin = padded element (h, ..., h)
    int64_t lin = 0;
    for (int d = 0; d < dim; ++d) lin = lin * v->pext[c][d] + halo;
    v->origin[c] = dst + lin * es;
  }
  CU(cudaStreamSynchronize(st));
  *out = v;
  return SG_OK;
}

int sg_volume_free(sg_volume* v) {
  if (!v) return SG_OK;
  cudaSetDevice(v->device);
  volume_textures_free(v);
  if (v->alloc) cudaFree(v->alloc);
  delete v;
  return SG_OK;
}

int sg_volume_bytes(const sg_volume* v, int64_t* bytes) {
  if (!v || !bytes) return fail(SG_EINVAL, "NULL argument");
  *bytes = (int64_t)v->bytes;
  return SG_OK;
}

int sg_volume_coset_ptr(const sg_volume* v, int coset, void** ptr) {
  if (!v || !ptr || coset < 0 || coset >= v->ncosets) return fail(SG_EINVAL, "bad argument");
  *ptr = (char*)v->alloc + v->coset_off[coset];
  return SG_OK;
}

int sg_volume_replicate(const sg_volume* v, int device, void* stream, sg_volume** out) {
  if (!v || !out) return fail(SG_EINVAL, "NULL argument");
  CU(cudaSetDevice(device));
  sg_volume* r = new sg_volume(*v);
  r->device = device;
  for (int c = 0; c < SG_MAX_COSETS; ++c) {   // textures are per volume: rebuilt on use
    r->tarr[c] = nullptr;
    r->tex[c] = 0;
  }
  r->tex_ready = false;
  cudaError_t e = cudaMalloc(&r->alloc, r->bytes);
  if (e != cudaSuccess) {
    delete r;
    return fail(SG_ENOMEM, "cudaMalloc: %s", cudaGetErrorString(e));
  }
  int can = 0;
  if (device != v->device) cudaDeviceCanAccessPeer(&can, device, v->device);
  if (device == v->device)
    e = cudaMemcpyAsync(r->alloc, v->alloc, r->bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
  else
    e = cudaMemcpyPeerAsync(r->alloc, device, v->alloc, v->device, r->bytes, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) {
    cudaFree(r->alloc);
    delete r;
    return fail(SG_ECUDA, "replicate: %s", cudaGetErrorString(e));
  }
  for (int c = 0; c < r->ncosets; ++c)
    r->origin[c] = (char*)r->alloc + ((const char*)v->origin[c] - (const char*)v->alloc);
  *out = r;
  return SG_OK;
}

static int check_pair(const sg_module* m, const sg_volume* v) {
  const sg_module_info& in = m->info;
  if (v->dim != in.dim) return fail(SG_EINVAL, "volume dim %d, kernel wants %d", v->dim, in.dim);
  if (v->ncosets != in.ncosets)
    return fail(SG_EINVAL, "data has %d cosets, program wants %d", v->ncosets, in.ncosets);
  if (v->dtype != in.dtype) return fail(SG_EINVAL, "volume dtype does not match the kernel");
  if (v->device != m->device) return fail(SG_EINVAL, "volume and module on different devices");
  if (v->halo != in.halo)
    return fail(SG_EINVAL, "volume halo %d, kernel compiled for %d", v->halo, in.halo);
  for (int c = 0; c < in.ncosets; ++c)
    for (int d = 0; d < in.dim; ++d)
      if (v->pext[c][d] != in.padded_extents[c][d])
        return fail(SG_EINVAL,
                    "coset %d axis %d: padded extent %lld, kernel compiled for %lld "
                    "(regenerate the program for this volume)",
                    c, d, (long long)v->pext[c][d], (long long)in.padded_extents[c][d]);
  return SG_OK;
}

// Counting sort of the queries by coset-0 cell bins into the module's scratch (caller holds
// bin_mu): sg_bin_count -> sg_bin_plan -> sg_bin_scatter_tiled.  Used by binned evaluation
// (bricks per bin) and by presort kernels (locality only).  The launch is ordered behind the
// module's previous one (bin_done); the caller records bin_done after its evaluation kernel.
static int sort_queries(sg_module* m, const void* xs, int64_t n, cudaStream_t st, float4** sorted_out,
                        int** starts_out, int2** items_out, long long* max_items_out) {
  const sg_module_info& in = m->info;
  const size_t nb = (size_t)m->nbins;
  if (nb > (size_t)SG_SMEM_BINS)
    return fail(SG_EINVAL, "%zu bins exceed the %d supported by the binning kernels; use a larger bin",
                nb, SG_SMEM_BINS);
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, m->device);
  // sort CTAs: `sort_ctas_per_sm` per SM (env SPLINEGPU_SORT_CTAS, default 2) of
  // `scatter_threads` threads (env SPLINEGPU_SCATTER_THREADS: 1024 | 512 | 256)
  static const int scatter_threads_env = [] {
    const char* e = getenv("SPLINEGPU_SCATTER_THREADS");
    const int v = e ? atoi(e) : 0;
    return (v == 256 || v == 512 || v == 1024) ? v : 0;
  }();
  static const long long min_per = [] {   // queries per sort CTA at least (env SPLINEGPU_SORT_MINPER)
    const char* e = getenv("SPLINEGPU_SORT_MINPER");
    const long long v = e ? atoll(e) : 8192;
    return v >= 1024 ? v : 8192;
  }();
  static const int sort_ctas_per_sm = [] {
    const char* e = getenv("SPLINEGPU_SORT_CTAS");
    const int v = e ? atoi(e) : 2;
    return v >= 1 && v <= 16 ? v : 2;
  }();
  const long long G = std::max<long long>(
      1, std::min<long long>((n + min_per - 1) / min_per, (long long)sort_ctas_per_sm * dev_sms));
  // measured on B200: long per-CTA ranges (>= 32K queries) scatter best with 512-thread
  // tiles, short ones with 1024-thread tiles (fewer barriers per query)
  const int scatter_threads = scatter_threads_env ? scatter_threads_env
                                                  : ((n + G - 1) / G >= 32768 ? 512 : 1024);
  static const int scatter_groups_env = [] {   // queries per thread / 4 (env SPLINEGPU_SCATTER_GROUPS)
    const char* e = getenv("SPLINEGPU_SCATTER_GROUPS");
    return e ? atoi(e) : 0;
  }();
  int scatter_groups = scatter_groups_env > 0 ? scatter_groups_env : 1;
  if (!((scatter_threads == 512 && scatter_groups == 2) || (scatter_threads == 256 && scatter_groups == 4)))
    scatter_groups = 1;
  const long long per = ((n + G - 1) / G + 3) & ~3LL;   // multiple of 4: float4 query groups
  const long long mlen = (long long)nb * G;
  const int chunk = std::max(32, in.chunk);
  const long long max_items = (n + chunk - 1) / chunk + (long long)nb;
  // layout: bin totals (kept zero between calls) | cursors | starts | count matrix | items | records
  const size_t head = ((3 * nb + 1) * sizeof(int) + 15) & ~(size_t)15;
  const size_t need = head + (((size_t)mlen * sizeof(int) + 15) & ~(size_t)15) +
                      (size_t)max_items * sizeof(int2) + (size_t)n * sizeof(float4) + 512;
  if (m->bin_scratch_bytes < need) {
    if (m->bin_scratch) cudaFree(m->bin_scratch);
    m->bin_scratch = nullptr;
    m->bin_scratch_bytes = 0;
    CU(cudaMalloc(&m->bin_scratch, need));
    CU(cudaMemset(m->bin_scratch, 0, head));
    m->bin_scratch_bytes = need;
  }
  int* bin_tot = (int*)m->bin_scratch;
  int* cursor = bin_tot + nb;
  int* starts = cursor + nb;
  int* mat = (int*)((char*)m->bin_scratch + head);
  int2* items = (int2*)((char*)mat + (((size_t)mlen * sizeof(int) + 15) & ~(size_t)15));
  float4* sorted = (float4*)(((uintptr_t)(items + max_items) + 255) & ~(uintptr_t)255);
  if (!m->bin_done) CU(cudaEventCreateWithFlags(&m->bin_done, cudaEventDisableTiming));
  CU(cudaStreamWaitEvent(st, m->bin_done, 0));   // the previous launch has released the scratch
  BinGeom g{};
  g.dim = in.dim;
  g.bin = in.bin;
  g.inv_bin = 1.0f / (float)in.bin;
  for (int d = 0; d < 3; ++d) {
    g.ext[d] = d < in.dim ? (float)in.extents[d] : 1.f;
    g.inv_ext[d] = 1.0f / g.ext[d];
    g.nb[d] = d < in.dim ? (int)m->nb[d] : 1;
  }
  g.nbins = (long long)nb;
  static std::once_flag attr_once;
  std::call_once(attr_once, [] {
    cudaFuncSetAttribute(sg_bin_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         2 * SG_SMEM_BINS * sizeof(int));
    cudaFuncSetAttribute(sg_bin_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         SG_SMEM_BINS * sizeof(int));
    const int tb = 4 * sg_tiled_max_bins() * sizeof(int);
    int optin = 227 * 1024;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
    auto attr = [&](const void* f, int recs) {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, f);
      const int cap = optin - (int)fa.sharedSizeBytes;   // dynamic + static <= the opt-in limit
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           std::min(cap, recs * (int)(sizeof(float4) + sizeof(int)) + tb));
    };
    attr((const void*)sg_bin_scatter_tiled<1024, 1>, 4096);
    attr((const void*)sg_bin_scatter_tiled<512, 1>, 2048);
    attr((const void*)sg_bin_scatter_tiled<512, 2>, 4096);
    attr((const void*)sg_bin_scatter_tiled<256, 1>, 1024);
    attr((const void*)sg_bin_scatter_tiled<256, 4>, 4096);
    cudaGetLastError();   // an attribute the device refuses shows up at launch, not here
  });
  sg_bin_count<<<(unsigned)G, SG_SORT_THREADS, nb * sizeof(int), st>>>((const float*)xs, (long long)n,
                                                                      per, g, mat, bin_tot);
  CU(cudaGetLastError());
  sg_bin_plan<<<1, 1024, 0, st>>>(bin_tot, (int)nb, (long long)n, chunk, starts, cursor, items,
                                  (int)max_items);
  CU(cudaGetLastError());
  const size_t shb = 4 * scatter_threads * scatter_groups * (sizeof(float4) + sizeof(int)) +
                     4 * nb * sizeof(int);
  int optin_now = 227 * 1024;
  cudaDeviceGetAttribute(&optin_now, cudaDevAttrMaxSharedMemoryPerBlockOptin, m->device);
  if (nb <= (size_t)sg_tiled_max_bins() && shb + 1024 <= (size_t)optin_now) {
    const float* xq = (const float*)xs;
    if (scatter_threads == 256 && scatter_groups == 4)
      sg_bin_scatter_tiled<256, 4><<<(unsigned)G, 256, shb, st>>>(xq, (long long)n, per, g, mat, cursor, sorted);
    else if (scatter_threads == 256)
      sg_bin_scatter_tiled<256, 1><<<(unsigned)G, 256, shb, st>>>(xq, (long long)n, per, g, mat, cursor, sorted);
    else if (scatter_threads == 512 && scatter_groups == 2)
      sg_bin_scatter_tiled<512, 2><<<(unsigned)G, 512, shb, st>>>(xq, (long long)n, per, g, mat, cursor, sorted);
    else if (scatter_threads == 512)
      sg_bin_scatter_tiled<512, 1><<<(unsigned)G, 512, shb, st>>>(xq, (long long)n, per, g, mat, cursor, sorted);
    else
      sg_bin_scatter_tiled<1024, 1><<<(unsigned)G, 1024, shb, st>>>(xq, (long long)n, per, g, mat, cursor, sorted);
  } else {
    sg_bin_scatter<<<(unsigned)G, SG_SORT_THREADS, nb * sizeof(int), st>>>(
        (const float*)xs, (long long)n, per, g, mat, cursor, sorted);
  }
  CU(cudaGetLastError());
  *sorted_out = sorted;
  *starts_out = starts;
  *items_out = items;
  *max_items_out = max_items;
  return SG_OK;
}

static int launch_binned(sg_module* m, const sg_volume* v, const void* xs, int64_t n, void* out,
                         void* grad, int32_t* dbg, cudaStream_t st) {
  const sg_module_info& in = m->info;
  std::lock_guard<std::mutex> lock(m->bin_mu);
  float4* sorted = nullptr;
  int* starts = nullptr;
  int2* items = nullptr;
  long long max_items = 0;
  int rc0 = sort_queries(m, xs, n, st, &sorted, &starts, &items, &max_items);
  if (rc0) return rc0;
  SgCosets cs{};
  for (int c = 0; c < v->ncosets; ++c) cs.base[c] = v->origin[c];
  static thread_local SgTmaps tm;
  memset(&tm, 0, sizeof tm);
  if (in.stage_tma) {
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return fail(SG_ECUDA, "cuTensorMapEncodeTiled is unavailable");
    for (int c = 0; c < v->ncosets; ++c) {
      cuuint64_t gdim[SG_MAX_DIM], gstr[SG_MAX_DIM];
      cuuint32_t box[SG_MAX_DIM], estr[SG_MAX_DIM];
      const int s = in.dim;
      long long stride = sizeof(float);
      for (int d = 0; d < s; ++d) {  // TMA dims are innermost-first
        const int ax = s - 1 - d;
        gdim[d] = (cuuint64_t)v->pext[c][ax];
        box[d] = (cuuint32_t)in.brick[ax];
        estr[d] = 1;
        if (d > 0) gstr[d - 1] = (cuuint64_t)stride;
        stride *= v->pext[c][ax];
      }
      void* gaddr = (char*)v->alloc + v->coset_off[c];
      CUresult r = enc(&tm.m[c], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)s, gaddr, gdim,
                       gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return fail(SG_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }
  }
  unsigned* err = nullptr;
  std::unique_lock<std::mutex> slot_lock;
  int slot = 0;
  int rc = acquire_slot(m, st, false, slot_lock, &slot, &err);
  if (rc) return rc;
  const void* sp = sorted;
  const void* stp = starts;
  const void* itp = items;
  void* args[] = {(void*)&sp, (void*)&stp, (void*)&itp, (void*)&out, (void*)&grad, (void*)&dbg,
                  (void*)&err, (void*)&cs, (void*)&tm};
  rc = timed_launch(m, (const void*)m->kernel, dim3((unsigned)max_items), dim3(in.block), args,
                    (size_t)in.smem_bytes, st);
  if (rc) return rc;
  rc = release_slot(m, slot, st);
  if (rc) return rc;
  CU(cudaEventRecord(m->bin_done, st));
  return SG_OK;
}

static int launch(sg_module* m, const sg_volume* v, const void* xs, int64_t n, void* out,
                  void* grad, int32_t* dbg, cudaStream_t st) {
  if (n <= 0) return SG_OK;
  // the query sort (binned and presort modules) keeps 32-bit query indices, bin starts and
  // cursors: batches of 2^30 or more queries are evaluated in 2^30-query pieces
  const int64_t kSortMax = (int64_t)1 << 30;
  if ((m->info.mode == SG_MODE_BINNED || m->info.presort) && n > kSortMax) {
    const size_t es = dtype_size(m->info.dtype);
    const int s = m->info.dim;
    for (int64_t q0 = 0; q0 < n; q0 += kSortMax) {
      const int64_t cnt = std::min(kSortMax, n - q0);
      int rc = launch(m, v, (const char*)xs + (size_t)q0 * s * es, cnt, (char*)out + (size_t)q0 * es,
                      grad ? (char*)grad + (size_t)q0 * s * es : nullptr,
                      dbg ? dbg + (size_t)q0 * m->info.ncosets * (s + 1) : nullptr, st);
      if (rc) return rc;
    }
    return SG_OK;
  }
  if (m->info.mode == SG_MODE_BINNED) return launch_binned(m, v, xs, n, out, grad, dbg, st);
  std::unique_lock<std::mutex> presort_lock;
  if (m->info.presort) {
    // locality pre-sort: the kernel reads (x, y, z, index) records in bin order
    presort_lock = std::unique_lock<std::mutex>(m->bin_mu);
    float4* sorted = nullptr;
    int* starts = nullptr;
    int2* items = nullptr;
    long long max_items = 0;
    int rc0 = sort_queries(m, xs, n, st, &sorted, &starts, &items, &max_items);
    if (rc0) return rc0;
    xs = sorted;
  }
  SgCosets cs{};
  for (int c = 0; c < v->ncosets; ++c) cs.base[c] = v->origin[c];
  SgTex tx{};
  const bool linear = m->info.mode == SG_MODE_LINEAR;
  if (linear) {
    int rt = volume_textures(const_cast<sg_volume*>(v), st);
    if (rt) return rt;
    for (int c = 0; c < v->ncosets; ++c) tx.t[c] = v->tex[c];
  }
  long long nn = (long long)n;
  unsigned* err = nullptr;
  void* args[] = {(void*)&xs, (void*)&nn, (void*)&out, (void*)&grad, (void*)&dbg, (void*)&err,
                  linear ? (void*)&tx : (void*)&cs};
  long long per_block = (long long)m->info.block * m->info.queries_per_thread;
  long long grid = (nn + per_block - 1) / per_block;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device);
  // grid-stride kernel: four waves of resident CTAs, so the per-CTA table staging is
  // amortized over many queries; kernels with dynamic shared memory (sorted tiles) run
  // one persistent wave
  long long cap = (long long)sms * std::max(1, 2048 / m->info.block) * 2;
  {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)m->kernel, m->info.block, 0) ==
            cudaSuccess && occ > 0)
      cap = (long long)sms * occ * 4;
    cudaGetLastError();
  }
  if (m->info.smem_bytes > 0) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)m->kernel, m->info.block,
                                                      (size_t)m->info.smem_bytes) != cudaSuccess ||
        occ < 1)
      occ = 1;
    cap = (long long)sms * occ;
  }
  grid = std::min(grid, cap);
  std::unique_lock<std::mutex> slot_lock;
  int slot = 0;
  // sorted kernels claim their tiles from the slot's counter
  int rc = acquire_slot(m, st, m->info.smem_bytes > 0, slot_lock, &slot, &err);
  if (rc) return rc;
  rc = timed_launch(m, (const void*)m->kernel, dim3((unsigned)grid), dim3(m->info.block), args,
                    (size_t)std::max(0, m->info.smem_bytes), st, v->alloc, v->bytes);
  if (rc) return rc;
  rc = release_slot(m, slot, st);
  if (rc) return rc;
  if (m->info.presort) CU(cudaEventRecord(m->bin_done, st));
  return SG_OK;
}

int sg_render(sg_module* m, const sg_volume* v, const float* rays, int64_t npix, int32_t steps,
              const float* tf, float* rgba, void* stream) {
  if (!m || !v) return fail(SG_EINVAL, "NULL module or volume");
  if (m->info.mode != SG_MODE_RENDER) return fail(SG_EINVAL, "module was not generated in render mode");
  if (npix < 0 || steps < 0) return fail(SG_EINVAL, "negative pixel or step count");
  if (npix == 0) return SG_OK;
  if (!rays || !tf || !rgba) return fail(SG_EINVAL, "NULL rays/tf/rgba");
  if (((uintptr_t)rays & 15) || ((uintptr_t)rgba & 15))
    return fail(SG_EINVAL, "rays and rgba must be 16-byte aligned");
  int rc = check_pair(m, v);
  if (rc) return rc;
  CU(cudaSetDevice(m->device));
  SgCosets cs{};
  for (int c = 0; c < v->ncosets; ++c) cs.base[c] = v->origin[c];
  long long nn = (long long)npix;
  int st = steps;
  unsigned* err = nullptr;
  void* args[] = {(void*)&rays, (void*)&nn, (void*)&rgba, (void*)&tf, (void*)&st, (void*)&err,
                  (void*)&cs};
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device);
  long long grid = (nn + m->info.block - 1) / m->info.block;
  grid = std::min(grid, (long long)sms * std::max(1, 2048 / m->info.block) * 4);
  if (m->info.smem_bytes > 0) {
    // psi-sorted renderer: persistent CTAs over blocks of 128 rays
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)m->kernel, m->info.block,
                                                      (size_t)m->info.smem_bytes) != cudaSuccess ||
        occ < 1)
      occ = 1;
    grid = std::min((nn + 127) / 128, (long long)sms * occ);
  }
  std::unique_lock<std::mutex> slot_lock;
  int slot = 0;
  // the psi-sorted renderer claims its ray blocks from the slot's counter
  rc = acquire_slot(m, (cudaStream_t)stream, m->info.smem_bytes > 0, slot_lock, &slot, &err);
  if (rc) return rc;
  rc = timed_launch(m, (const void*)m->kernel, dim3((unsigned)grid), dim3(m->info.block), args,
                    (size_t)std::max(0, m->info.smem_bytes), (cudaStream_t)stream, v->alloc,
                    v->bytes);
  if (rc) return rc;
  return release_slot(m, slot, (cudaStream_t)stream);
}

int sg_eval(sg_module* m, const sg_volume* v, const void* xs, int64_t n, void* out, void* grad,
            int32_t* dbg, void* stream) {
  if (!m || !v) return fail(SG_EINVAL, "NULL module or volume");
  if (m->info.mode == SG_MODE_RENDER) return fail(SG_EINVAL, "render-mode modules are launched with sg_render");
  if (n < 0) return fail(SG_EINVAL, "negative point count");
  if (n > 0 && (!xs || !out)) return fail(SG_EINVAL, "NULL xs/out");
  if (m->info.has_dbg && n > 0 && !dbg) return fail(SG_EINVAL, "kernel writes dbg; pass a buffer");
  if (m->info.has_grad && n > 0 && !grad) return fail(SG_EINVAL, "kernel writes grad; pass a buffer");
  int rc = check_pair(m, v);
  if (rc) return rc;
  CU(cudaSetDevice(m->device));
  return launch(m, v, xs, n, out, grad, dbg, (cudaStream_t)stream);
}

int sg_eval_host(sg_module* m, const sg_volume* v, const void* xs_host, int64_t n,
                 void* out_host, void* grad_host, int64_t chunk) {
  if (!m || !v) return fail(SG_EINVAL, "NULL module or volume");
  if (n < 0) return fail(SG_EINVAL, "negative point count");
  if (n == 0) return SG_OK;
  if (!xs_host || !out_host) return fail(SG_EINVAL, "NULL xs/out");
  if (m->info.has_dbg) return fail(SG_EINVAL, "debug kernels are device-path only");
  if (m->info.mode == SG_MODE_RENDER) return fail(SG_EINVAL, "render-mode modules are launched with sg_render");
  if (m->info.has_grad && !grad_host) return fail(SG_EINVAL, "kernel writes grad; pass a buffer");
  int rc = check_pair(m, v);
  if (rc) return rc;
  std::lock_guard<std::mutex> lock(m->mu);
  CU(cudaSetDevice(m->device));
  const int s = m->info.dim;
  const size_t es = dtype_size(m->info.dtype);
  // default chunk: 2^21 queries, but at least 4 chunks down to 2^18 so small batches still
  // overlap H2D, kernel and D2H (measured on B200: c1's 2^20 queries 2.57 -> 2.84 G/s e2e)
  if (chunk <= 0) chunk = std::min<int64_t>(1 << 21, std::max<int64_t>(1 << 18, n / 4));
  chunk = std::min<int64_t>(chunk, n);
  const int nst = 3;
  const size_t per_pt = es * (s + 1 + (m->info.has_grad ? s : 0));
  const size_t need = (size_t)chunk * per_pt * nst;
  if (m->scratch_bytes < need) {
    if (m->scratch) cudaFree(m->scratch);
    m->scratch = nullptr;
    m->scratch_bytes = 0;
    CU(cudaMalloc(&m->scratch, need));
    m->scratch_bytes = need;
  }
  for (auto& st : m->streams)
    if (!st) CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  for (int64_t start = 0, it = 0; start < n; start += chunk, ++it) {
    const int64_t cnt = std::min<int64_t>(chunk, n - start);
    const int k = (int)(it % nst);
    cudaStream_t st = m->streams[k];
    char* base = (char*)m->scratch + (size_t)k * chunk * per_pt;
    char* dxs = base;
    char* dout = dxs + (size_t)chunk * es * s;
    char* dgrad = m->info.has_grad ? dout + (size_t)chunk * es : nullptr;
    CU(cudaMemcpyAsync(dxs, (const char*)xs_host + (size_t)start * s * es, (size_t)cnt * s * es,
                       cudaMemcpyHostToDevice, st));
    rc = launch(m, v, dxs, cnt, dout, dgrad, nullptr, st);
    if (rc) return rc;
    CU(cudaMemcpyAsync((char*)out_host + (size_t)start * es, dout, (size_t)cnt * es,
                       cudaMemcpyDeviceToHost, st));
    if (dgrad)
      CU(cudaMemcpyAsync((char*)grad_host + (size_t)start * s * es, dgrad, (size_t)cnt * s * es,
                         cudaMemcpyDeviceToHost, st));
  }
  for (auto& st : m->streams) CU(cudaStreamSynchronize(st));
  return SG_OK;
}

}  // extern "C"
