// whff_common.cuh -- device pieces shared by the translation units of
// libwhff_b200.so (whff_b200.cu, whff_packed.cu): the device view of a WHFZ
// stream, segment location, the any-layout block decoder entry, the inverse
// lift matrix G and the block-column vector slice.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "../../include/whff_b200.h"
#include "whff_decode.cuh"
#include "whff_relayout.cuh"

using namespace whff;

// Opt a kernel into more than 48 KB of dynamic shared memory, once per
// device (the attribute belongs to the function's instance in the current
// device's context).  `done` is the kernel's own per-device bitmask.
template <typename Kernel>
static cudaError_t ensure_dyn_smem(Kernel* k, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// ---------------------------------------------------------------------------
// device view of a stream
// ---------------------------------------------------------------------------
struct StreamView {
  const uint32_t* words;     // payload as LE uint32 words (padded)
  const uint64_t* base;      // COMPACT: start bit of block (br, 32g)
  const uint16_t* lens;      // COMPACT/FULL: segment bits (clamped 65535)
  const uint64_t* starts;    // FULL: start bit per block
  uint64_t payload_bits;
  uint64_t rows, cols, br, bc, gpr;
  uint32_t seg_bits;         // IMPLICIT: 16 * bpv
  int32_t kind;
  int32_t planes_limit;
  int32_t has_raw;
  int32_t layout;
};

__device__ __forceinline__ int clamp_len(uint64_t start, uint64_t seg, uint64_t payload_bits) {
  if (start >= payload_bits) return 0;
  uint64_t lim = start + seg;
  if (lim > payload_bits) lim = payload_bits;
  const uint64_t l = lim - start;
  return l > 65535u ? 65535 : (int)l;
}

// start/len of one block, any index kind (COMPACT walks <= 31 lengths)
static __device__ void block_extent(const StreamView& s, uint64_t b, uint64_t& start, int& len) {
  if (s.kind == WHFF_INDEX_IMPLICIT) {
    start = b * (uint64_t)s.seg_bits;
    len = clamp_len(start, s.seg_bits, s.payload_bits);
  } else if (s.kind == WHFF_INDEX_FULL) {
    start = s.starts[b];
    len = clamp_len(start, s.lens[b], s.payload_bits);
  } else {
    const uint64_t brow = b / s.bc, bcol = b % s.bc;
    const uint64_t g0 = bcol & ~31ull;
    uint64_t st = s.base[brow * s.gpr + (bcol >> 5)];
    for (uint64_t c = g0; c < bcol; ++c) st += s.lens[brow * s.bc + c];
    start = st;
    len = clamp_len(start, s.lens[b], s.payload_bits);
  }
}

// either layout, refill path, for the thread-per-block kernels
template <bool HAS_RAW>
__device__ __forceinline__ void decode_any(const StreamView& s, BitWin& bw, int planes_limit,
                                           Decoded& d) {
  if (s.layout == WHFF_LAYOUT_SKELETON_FIRST)
    decode_block_sf<HAS_RAW, true>(bw, planes_limit, d);
  else
    decode_block<HAS_RAW, true>(bw, planes_limit, d, __activemask());
}

// G = real-valued inverse lift (codec.py:128-134 with >>1 -> /2, <<1 -> *2);
// the decoded block is 2^(e-26) * G Q G^T up to lift rounding.
static __device__ __constant__ float c_G[4][4] = {{1.0f, 1.5f, -1.0f, -0.25f},
                                          {1.0f, 0.5f, 1.0f, 1.25f},
                                          {1.0f, -0.5f, 1.0f, -1.25f},
                                          {1.0f, -1.5f, -1.0f, 0.25f}};

// block-column vector slice, zero padded past cols
__device__ __forceinline__ float4 load_v4(const float* v, uint64_t bcol, uint64_t cols, bool aligned) {
  const uint64_t c0 = bcol * 4;
  if (aligned && c0 + 3 < cols) return ldg(reinterpret_cast<const float4*>(v) + bcol);
  float4 r;
  r.x = c0 + 0 < cols ? ldg(v + c0 + 0) : 0.0f;
  r.y = c0 + 1 < cols ? ldg(v + c0 + 1) : 0.0f;
  r.z = c0 + 2 < cols ? ldg(v + c0 + 2) : 0.0f;
  r.w = c0 + 3 < cols ? ldg(v + c0 + 3) : 0.0f;
  return r;
}


// A block-row's (band's) column groups are summed in kVW "virtual warps"
// (see k_decode_gemv / k_pk_gemv).
constexpr int kVW = 32;
