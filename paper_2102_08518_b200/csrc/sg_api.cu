// sg_api.cu -- implementation of include/splinegpu.h (the C-ABI boundary).
//
// Built with nvcc for sm_100a into libsplinegpu.so.  The CUDA runtime is linked
// statically (no libcuda link-time dependency, so the library loads -- and its
// symbols can be checked -- on a machine without a GPU); NVRTC is linked
// dynamically from the image's CUDA 12.9 toolkit.  Generated kernels are loaded
// with the context-independent library API (cudaLibraryLoadData) and launched
// with cudaLaunchKernel, so no driver-API symbols are needed.
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

}  // namespace

struct sg_module {
  int device = 0;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kernel = nullptr;
  sg_module_info info{};
  unsigned* d_err = nullptr;
  int regs = 0, local_bytes = 0;
  std::mutex mu;  // guards the host-path scratch below
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  cudaStream_t streams[3] = {nullptr, nullptr, nullptr};
};

struct sg_volume {
  int device = 0;
  int dim = 0, ncosets = 0, halo = 0, dtype = SG_F32;
  int64_t ext[SG_MAX_COSETS][SG_MAX_DIM] = {};
  int64_t pext[SG_MAX_COSETS][SG_MAX_DIM] = {};
  void* alloc = nullptr;  // one allocation, coset-split
  size_t bytes = 0;
  size_t coset_off[SG_MAX_COSETS] = {};  // byte offset of each coset's padded array
  const void* origin[SG_MAX_COSETS] = {};  // padded element (h, h, ..., h)
};

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
  (void)image_len;
  if (!image || !entry || !info || !out) return fail(SG_EINVAL, "NULL argument");
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
  e = cudaMalloc(&m->d_err, sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemset(m->d_err, 0, sizeof(unsigned));
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
  if (m->d_err) cudaFree(m->d_err);
  if (m->lib) cudaLibraryUnload(m->lib);
  delete m;
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
  unsigned h = 0;
  cudaStream_t st = (cudaStream_t)stream;
  CU(cudaMemcpyAsync(&h, m->d_err, sizeof h, cudaMemcpyDeviceToHost, st));
  CU(cudaMemsetAsync(m->d_err, 0, sizeof h, st));
  CU(cudaStreamSynchronize(st));
  if (flags) *flags = h;
  if (h & 1u) return fail(SG_EUNREACHABLE, "point classified into an unreachable sigma entry");
  return SG_OK;
}

int sg_volume_create(int device, int dim, int ncosets, const int64_t* extents, int halo,
                     int dtype, const void* const* src, int src_on_device, void* stream,
                     sg_volume** out) {
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
      v->pext[c][d] = e + 2 * halo;
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
  for (int c = 0; c < in.ncosets; ++c)
    for (int d = 0; d < in.dim; ++d)
      if (v->pext[c][d] != in.padded_extents[c][d])
        return fail(SG_EINVAL,
                    "coset %d axis %d: padded extent %lld, kernel compiled for %lld "
                    "(regenerate the program for this volume)",
                    c, d, (long long)v->pext[c][d], (long long)in.padded_extents[c][d]);
  return SG_OK;
}

static int launch(sg_module* m, const sg_volume* v, const void* xs, int64_t n, void* out,
                  void* grad, int32_t* dbg, cudaStream_t st) {
  if (n <= 0) return SG_OK;
  SgCosets cs{};
  for (int c = 0; c < v->ncosets; ++c) cs.base[c] = v->origin[c];
  long long nn = (long long)n;
  unsigned* err = m->d_err;
  void* args[] = {(void*)&xs, (void*)&nn, (void*)&out, (void*)&grad, (void*)&dbg, (void*)&err,
                  (void*)&cs};
  long long per_block = (long long)m->info.block * m->info.queries_per_thread;
  long long grid = (nn + per_block - 1) / per_block;
  if (grid > 0x7fffffffLL) return fail(SG_EINVAL, "batch too large for one launch");
  CU(cudaLaunchKernel((const void*)m->kernel, dim3((unsigned)grid), dim3(m->info.block), args, 0,
                      st));
  return SG_OK;
}

int sg_eval(sg_module* m, const sg_volume* v, const void* xs, int64_t n, void* out, void* grad,
            int32_t* dbg, void* stream) {
  if (!m || !v) return fail(SG_EINVAL, "NULL module or volume");
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
  if (m->info.has_grad && !grad_host) return fail(SG_EINVAL, "kernel writes grad; pass a buffer");
  int rc = check_pair(m, v);
  if (rc) return rc;
  std::lock_guard<std::mutex> lock(m->mu);
  CU(cudaSetDevice(m->device));
  const int s = m->info.dim;
  const size_t es = dtype_size(m->info.dtype);
  if (chunk <= 0) chunk = 1 << 21;
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
