/*
 * whff_gemv_file.c -- a non-Python host of the C ABI (include/whff_b200.h).
 *
 * Reads a WHFZ stream file (the reference's container, codec.py:388-450 /
 * "WHFZ", u16 version, u8 mode, u32|f64 param, u64 rows,
 * u64 cols, u8 block, u64 n_blocks, u64 index[n_blocks], payload), uploads it,
 * switches it to the skeleton-first device layout and computes y = C v with
 * v = 1 (or v_j = (j % 7 + 1) / 8 with --ramp) through the fused
 * decode + GEMV, printing one line: rows, sum(y), y[0], y[rows-1].
 *
 * Build: gcc -O2 -I include -o whff_gemv_file examples/whff_gemv_file.c \
 *          -L paper_1902_08018_b200 -lwhff_b200 -L /usr/local/cuda/lib64 -lcudart
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "whff_b200.h"

#define CHECK(x)                                                                 \
  do {                                                                           \
    whff_status_t st_ = (x);                                                     \
    if (st_ != WHFF_OK) {                                                        \
      fprintf(stderr, "%s: %s (%s)\n", #x, whff_status_string(st_), whff_last_error()); \
      return 2;                                                                  \
    }                                                                            \
  } while (0)

static int rd(FILE* f, void* p, size_t n) { return fread(p, 1, n, f) == n ? 0 : -1; }

int main(int argc, char** argv) {
  if (argc < 2) {
    fprintf(stderr, "usage: %s stream.whfz [--coefficient] [--ramp]\n", argv[0]);
    return 1;
  }
  int eval = WHFF_EVAL_EXACT, ramp = 0;
  for (int i = 2; i < argc; ++i) {
    if (!strcmp(argv[i], "--coefficient")) eval = WHFF_EVAL_COEFF;
    if (!strcmp(argv[i], "--ramp")) ramp = 1;
  }
  FILE* f = fopen(argv[1], "rb");
  if (!f) { perror(argv[1]); return 1; }
  char magic[4];
  uint16_t version;
  uint8_t mode, block;
  uint64_t rows, cols, nb;
  double param = 0.0;
  if (rd(f, magic, 4) || memcmp(magic, "WHFZ", 4) || rd(f, &version, 2) || rd(f, &mode, 1)) {
    fprintf(stderr, "not a WHFZ stream\n");
    return 3;
  }
  if (mode == WHFF_MODE_ACCURACY) {
    if (rd(f, &param, 8)) return 3;
  } else {
    uint32_t p;
    if (rd(f, &p, 4)) return 3;
    param = p;
  }
  if (rd(f, &rows, 8) || rd(f, &cols, 8) || rd(f, &block, 1) || rd(f, &nb, 8)) return 3;
  uint64_t* index = malloc(nb * 8);
  if (!index || rd(f, index, nb * 8)) return 3;
  long here = ftell(f);
  fseek(f, 0, SEEK_END);
  const uint64_t payload_bytes = (uint64_t)(ftell(f) - here);
  fseek(f, here, SEEK_SET);
  uint8_t* payload = malloc(payload_bytes ? payload_bytes : 1);
  if (!payload || rd(f, payload, payload_bytes)) return 3;
  fclose(f);

  whff_dstream_t s;
  CHECK(whff_dstream_create(0, mode, param, rows, cols, payload, payload_bytes, index, nb, &s));
  CHECK(whff_dstream_relayout(s, WHFF_LAYOUT_SKELETON_FIRST, NULL));

  float *v_dev, *y_dev;
  uint64_t* status_dev;
  void* ws = NULL;
  size_t ws_bytes = 0;
  float* v = malloc(cols * sizeof(float));
  float* y = malloc(rows * sizeof(float));
  for (uint64_t j = 0; j < cols; ++j) v[j] = ramp ? (float)(j % 7 + 1) / 8.0f : 1.0f;
  CHECK(whff_decode_gemv_workspace_size(s, eval, &ws_bytes));
  if (cudaMalloc((void**)&v_dev, cols * 4) || cudaMalloc((void**)&y_dev, rows * 4) ||
      cudaMalloc((void**)&status_dev, 8) || (ws_bytes && cudaMalloc(&ws, ws_bytes)))
    return 4;
  const uint64_t clear = WHFF_STATUS_CLEAR;
  cudaMemcpy(v_dev, v, cols * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(status_dev, &clear, 8, cudaMemcpyHostToDevice);
  CHECK(whff_decode_gemv(s, v_dev, y_dev, WHFF_POLICY_MIXED, eval, 0, rows, ws, ws_bytes,
                         status_dev, NULL));
  uint64_t status;
  cudaMemcpy(y, y_dev, rows * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&status, status_dev, 8, cudaMemcpyDeviceToHost);
  if (status != WHFF_STATUS_CLEAR) {
    fprintf(stderr, "non-finite decoded value at flat index %llu\n", (unsigned long long)status);
    return 5;
  }
  double sum = 0.0;
  for (uint64_t i = 0; i < rows; ++i) sum += y[i];
  printf("%llu %.17g %.9g %.9g\n", (unsigned long long)rows, sum, y[0], y[rows - 1]);
  CHECK(whff_dstream_destroy(s));
  cudaFree(v_dev);
  cudaFree(y_dev);
  cudaFree(status_dev);
  if (ws) cudaFree(ws);
  free(v);
  free(y);
  free(index);
  free(payload);
  return 0;
}
