/*
 * splinegpu.h -- C ABI of the B200 (sm_100a) spline-reconstruction evaluator.
 *
 * This is the drop-in boundary for the reference's native execution path:
 * the reference lowers a spline space to LLVM IR, builds it with clang and calls
 *
 *     T reconstruct(T x0, ..., T x{s-1},
 *                   T* coset0, i64 ext0_0 ... ext0_{s-1}, ..., T* coset{M-1}, ...)
 *
 * once per query point through ctypes (reference pkg/src/splinegen/emit.py:237-241,
 * argtypes pkg/src/splinegen/bench.py:239-247, per-point loop bench.py:259-263).
 * Here the same computation is one batched, asynchronous launch over N points:
 *
 *   sg_compile        replaces `clang -O2 -shared kernel.ll` (bench.py:221-247): NVRTC
 *                     compiles the generated CUDA source for sm_100a to a cubin.
 *   sg_module_load    replaces ctypes.CDLL(kernel.so).reconstruct (bench.py:238).
 *   sg_volume_create  replaces the per-call (pointer, extents) pairs (bench.py:253-258):
 *                     coset arrays in the reference's C order (`DataVolume`,
 *                     ir.py:524-558) are uploaded once, with a periodic ghost halo, so
 *                     the per-fetch `srem` wrap of emit.py:186-212 happens once per coset.
 *   sg_eval           replaces the per-point `fn(*row, *fixed)` loop (bench.py:259-263):
 *                     xs is (N, s) row-major like `interpret_batch`'s input (ir.py:582).
 *   sg_eval_host      the same with HOST buffers: H2D, kernel and D2H pipelined over
 *                     chunks on internal streams (the end-to-end user call).
 *   sg_module_status  reads/clears the device error word; SG_EUNREACHABLE mirrors the
 *                     reference's sigma == -1 errors (ir.py:757-766, oracle.py:69-73),
 *                     which the LLVM path leaves undefined (emit.py:161-164).
 *
 * Ownership: the caller owns xs/out/grad/dbg (device pointers for sg_eval, host
 * pointers for sg_eval_host); the library owns modules and volumes.  All calls are
 * thread-safe per (module, stream); a binned module owns one sort scratch, so its
 * launches on different streams are ordered behind one another (an event per module)
 * while the host path's copies still overlap.  The only global mutable state is the
 * thread-local error string.  Every entry point returns an SG_* status.
 */
#ifndef SPLINEGPU_H
#define SPLINEGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SG_OK = 0,
  SG_EINVAL = 1,        /* shape / dtype / coset-count mismatch (ir.py:591-596) */
  SG_ECUDA = 2,         /* CUDA runtime error (message in sg_last_error) */
  SG_EUNREACHABLE = 3,  /* a point hit a sigma entry marked -1 */
  SG_ECOMPILE = 4,      /* NVRTC compilation failed (log in sg_last_error) */
  SG_ENOMEM = 5
};

enum { SG_F32 = 0, SG_F64 = 1 };

#define SG_MAX_COSETS 8
#define SG_MAX_DIM 4

typedef struct sg_module sg_module;
typedef struct sg_volume sg_volume;

/* Static description of a generated kernel, filled in by the code generator. */
typedef struct sg_module_info {
  int32_t dim;                 /* s, 1..4 */
  int32_t ncosets;             /* M, 1..SG_MAX_COSETS */
  int32_t dtype;               /* SG_F32 | SG_F64: volume, query and output type */
  int32_t block;               /* threads per CTA */
  int32_t has_grad;            /* kernel writes grad (N, s) */
  int32_t has_dbg;             /* kernel writes dbg (N, M, s+1): k then sub-region */
  int32_t halo;                /* padded index of interior element 0 on every axis */
  int32_t queries_per_thread;  /* >= 1 */
  int64_t padded_extents[SG_MAX_COSETS][SG_MAX_DIM]; /* per coset allocation extents */
  /* binned mode (SG_MODE_BINNED): queries are counting-sorted into bins of
   * `bin` lattice cells of coset 0; one CTA per bin stages the bin's coefficient
   * bricks (all cosets) in shared memory -- by TMA when stage_tma -- and gathers
   * from there.  Direct mode gathers through L1/L2. */
  int32_t mode;                /* SG_MODE_DIRECT | SG_MODE_BINNED */
  int32_t rounding;            /* coset-0 region map: SG_FLOOR | SG_ROUND */
  int32_t stage_tma;           /* 1: bricks staged with cp.async.bulk.tensor */
  int32_t smem_bytes;          /* dynamic shared memory of the binned kernel */
  int32_t bin;                 /* bin edge, in lattice cells */
  int32_t brick[SG_MAX_DIM];   /* brick extent per axis (elements), C order */
  int64_t extents[SG_MAX_DIM]; /* unpadded extents (equal for all cosets in binned mode) */
  int32_t chunk;               /* binned: queries per CTA work item */
  int32_t static_smem;         /* informational: static shared memory of the kernel */
  /* direct-mode kernels generated with presort: the library first counting-sorts the
   * queries by cubes of `bin` cells (the binned-mode sort, for locality only) and the
   * kernel reads the (x, y, z, original index) records, writing results by index */
  int32_t presort;
} sg_module_info;

/* SG_MODE_LINEAR: tensor-product kernels that fetch
 * pairs of neighbouring coefficients with ONE hardware-filtered texture read.  The library
 * binds one f32 texture per coset (cudaArray copy of the volume, wrap addressing, linear
 * filtering), built on the first launch against a volume; 8-bit filter weights make the
 * results ~1e-3 accurate -- opt-in, never the default. */
enum { SG_MODE_DIRECT = 0, SG_MODE_BINNED = 1, SG_MODE_RENDER = 2, SG_MODE_LINEAR = 3 };
enum { SG_FLOOR = 0, SG_ROUND = 1 };

int sg_version(void);
const char* sg_last_error(void);
int sg_device_count(int* count);

/* NVRTC: CUDA C++ source -> cubin for sm_100a.  *image is malloc'ed by the library
 * (release with sg_free).  opts may be NULL.  On SG_ECOMPILE the log is in
 * sg_last_error(). */
int sg_compile(const char* source, const char* name, const char* const* opts, int nopts,
               void** image, size_t* image_len, char** log);
void sg_free(void* p);

int sg_module_load(const void* image, size_t image_len, const char* entry, int device,
                   const sg_module_info* info, sg_module** out);
int sg_module_free(sg_module* m);
int sg_module_regs(const sg_module* m, int* regs_per_thread, int* local_bytes);
/* Reads the device error word (after synchronizing `stream`) and clears it.
 * Returns SG_EUNREACHABLE if any point hit sigma == -1 since the last call. */
int sg_module_status(sg_module* m, void* stream, uint32_t* flags);

/* Kernel timing for roofline reporting: while enabled, sg_eval brackets the evaluation
 * kernel (not the binning kernels) with CUDA events on the launch stream;
 * sg_module_kernel_time synchronizes them and returns the summed milliseconds and the
 * number of launches since the last call (then resets). */
int sg_module_timing(sg_module* m, int enable);
int sg_module_kernel_time(sg_module* m, double* total_ms, int64_t* launches);

/* extents: ncosets x dim (row-major); src[c] points to coset c's C-order array of
 * prod(extents[c]) elements, in HOST memory (src_on_device == 0) or device memory.
 * The device copy is periodic: padded element i holds src[(i - halo) mod E] on every
 * axis; padded (ncosets x dim, may be NULL = E + 2*halo) gives the allocation extents
 * a module asks for (sg_module_info.padded_extents). */
int sg_volume_create(int device, int dim, int ncosets, const int64_t* extents, int halo,
                     const int64_t* padded, int dtype, const void* const* src,
                     int src_on_device, void* stream, sg_volume** out);
int sg_volume_free(sg_volume* v);
int sg_volume_bytes(const sg_volume* v, int64_t* bytes);
/* Device address of coset c's padded array origin (for tests / peer copies). */
int sg_volume_coset_ptr(const sg_volume* v, int coset, void** ptr);

/* Asynchronous batched evaluation on `stream` (cudaStream_t; NULL = legacy default).
 * xs: n x dim row-major (device), out: n (device), grad: n x dim or NULL,
 * dbg: n x ncosets x (dim+1) int32 or NULL (required iff the module has_dbg). */
int sg_eval(sg_module* m, const sg_volume* v, const void* xs, int64_t n, void* out,
            void* grad, int32_t* dbg, void* stream);

/* End-to-end evaluation with HOST buffers: the library pipelines H2D(xs chunk),
 * kernel, D2H(out chunk) over `chunk` points per stage (0 = default) on its own
 * streams and returns after the results are on the host.  Pinned host memory is
 * recommended for full PCIe / C2C bandwidth. */
int sg_eval_host(sg_module* m, const sg_volume* v, const void* xs_host, int64_t n,
                 void* out_host, void* grad_host, int64_t chunk);

/* Fused volume rendering (SG_MODE_RENDER modules): the caller of the evaluation path in
 * the paper's application -- ray march, reconstruction (+ gradient shading)
 * and front-to-back compositing in one kernel, so samples never round-trip through HBM.
 * rays: npix x 8 floats (origin xyz, direction xyz, t0, dt), 16-B aligned, device memory;
 * sample j of a ray sits at o + (t0 + (j + 1/2) dt) d (fp32, round-to-nearest, no FMA).
 * tf: 12 floats (f_lo, 1/(f_hi - f_lo), opacity per unit length, rgb at f_lo, rgb at f_hi,
 * light direction xyz -- used when the module was generated with gradients).
 * rgba: npix x 4 floats (premultiplied colour, opacity). */
int sg_render(sg_module* m, const sg_volume* v, const float* rays, int64_t npix, int32_t steps,
              const float* tf, float* rgba, void* stream);

/* Replicate a volume onto other devices (peer copy over NVLink when available). */
int sg_volume_replicate(const sg_volume* v, int device, void* stream, sg_volume** out);

#ifdef __cplusplus
}
#endif
#endif /* SPLINEGPU_H */
