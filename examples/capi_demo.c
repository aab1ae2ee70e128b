/* Plain-C use of the drop-in boundary (include/splinegpu.h), no Python or torch:
 *
 *   capi_demo <kernel.cu> <info.txt> <volume.bin> <queries.bin> <out.bin>
 *
 * kernel.cu  generated CUDA source (paper_2102_08518_b200.cudagen.generate(...).source)
 * info.txt   "dim ncosets block halo mode rounding stage_tma smem bin chunk" then per coset
 *            the padded extents, then the unpadded extents and the brick
 * volume.bin ncosets x prod(extents) float32, C order per coset (the reference DataVolume)
 * queries.bin n x dim float32
 * out.bin    n float32 results (written)
 *
 * It is what a C / cgo / JNI caller of the reference's `reconstruct` (emit.py:237-241)
 * would do instead of calling it once per point: compile once, upload the volume once,
 * evaluate a batch through the pipelined host path. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/splinegpu.h"

static void* slurp(const char* path, size_t* len) {
  FILE* f = fopen(path, "rb");
  if (!f) { perror(path); exit(2); }
  fseek(f, 0, SEEK_END);
  *len = (size_t)ftell(f);
  fseek(f, 0, SEEK_SET);
  char* buf = (char*)malloc(*len + 1);
  if (fread(buf, 1, *len, f) != *len) { perror("read"); exit(2); }
  buf[*len] = 0;
  fclose(f);
  return buf;
}

#define CHECK(call)                                                          \
  do {                                                                       \
    int rc_ = (call);                                                        \
    if (rc_ != SG_OK) {                                                      \
      fprintf(stderr, "%s -> %d: %s\n", #call, rc_, sg_last_error());       \
      return 1;                                                              \
    }                                                                        \
  } while (0)

int main(int argc, char** argv) {
  if (argc != 6) {
    fprintf(stderr, "usage: %s kernel.cu info.txt volume.bin queries.bin out.bin\n", argv[0]);
    return 2;
  }
  size_t src_len, vol_len, q_len, info_len;
  char* src = (char*)slurp(argv[1], &src_len);
  char* info_txt = (char*)slurp(argv[2], &info_len);
  float* vol = (float*)slurp(argv[3], &vol_len);
  float* xs = (float*)slurp(argv[4], &q_len);

  sg_module_info info;
  memset(&info, 0, sizeof info);
  char* p = info_txt;
  info.dim = (int)strtol(p, &p, 10);
  info.ncosets = (int)strtol(p, &p, 10);
  info.block = (int)strtol(p, &p, 10);
  info.halo = (int)strtol(p, &p, 10);
  info.mode = (int)strtol(p, &p, 10);
  info.rounding = (int)strtol(p, &p, 10);
  info.stage_tma = (int)strtol(p, &p, 10);
  info.smem_bytes = (int)strtol(p, &p, 10);
  info.bin = (int)strtol(p, &p, 10);
  info.chunk = (int)strtol(p, &p, 10);
  info.dtype = SG_F32;
  info.queries_per_thread = 1;
  for (int c = 0; c < info.ncosets; ++c)
    for (int d = 0; d < info.dim; ++d) info.padded_extents[c][d] = strtoll(p, &p, 10);
  int64_t ext[SG_MAX_DIM];
  int64_t nel = 1;
  for (int d = 0; d < info.dim; ++d) {
    ext[d] = strtoll(p, &p, 10);
    info.extents[d] = ext[d];
    nel *= ext[d];
  }
  for (int d = 0; d < info.dim; ++d) info.brick[d] = (int)strtol(p, &p, 10);

  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17"};
  void* image = NULL;
  size_t image_len = 0;
  char* log = NULL;
  CHECK(sg_compile(src, "demo.cu", opts, 2, &image, &image_len, &log));
  sg_free(log);
  sg_module* mod = NULL;
  CHECK(sg_module_load(image, image_len, "sg_eval_kernel", 0, &info, &mod));

  int64_t exts[SG_MAX_COSETS * SG_MAX_DIM];
  const void* srcs[SG_MAX_COSETS];
  for (int c = 0; c < info.ncosets; ++c) {
    for (int d = 0; d < info.dim; ++d) exts[c * info.dim + d] = ext[d];
    srcs[c] = vol + (size_t)c * nel;
  }
  sg_volume* v = NULL;
  int64_t padded[SG_MAX_COSETS * SG_MAX_DIM];   /* ncosets x dim, packed */
  for (int c = 0; c < info.ncosets; ++c)
    for (int d = 0; d < info.dim; ++d) padded[c * info.dim + d] = info.padded_extents[c][d];
  CHECK(sg_volume_create(0, info.dim, info.ncosets, exts, info.halo, padded, SG_F32, srcs, 0, NULL,
                         &v));
  const int64_t n = (int64_t)(q_len / sizeof(float) / info.dim);
  float* out = (float*)malloc((size_t)n * sizeof(float));
  CHECK(sg_eval_host(mod, v, xs, n, out, NULL, 0));
  uint32_t flags = 0;
  CHECK(sg_module_status(mod, NULL, &flags));
  FILE* f = fopen(argv[5], "wb");
  fwrite(out, sizeof(float), (size_t)n, f);
  fclose(f);
  printf("capi_demo: %lld reconstructions, first %.9g\n", (long long)n, out[0]);
  sg_volume_free(v);
  sg_module_free(mod);
  sg_free(image);
  free(out);
  free(src);
  free(info_txt);
  free(vol);
  free(xs);
  return 0;
}
