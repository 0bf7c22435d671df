// whff_encode.cuh -- WHFZ block encoder (GPU `codec.compress`), one block per
// thread.  Byte-identical restatement of
//   whff/codec.py:157-164 (_to_blocks, edge replication), :186-198
//   (_block_exponents, _quantize), :118-125/:137-142 (_fwd_lift,
//   _forward_transform), :225-268 (compress), :271-293 (_select_planes),
//   whff/_kernels.pyx:139-225 (_encode_one) and :228-283 (encode_blocks).
// __host__ __device__ so tests can check it on the CPU (tools/hostcheck.cpp).
#pragma once
#include <math.h>
#include <stdint.h>
#include "whff_decode.cuh"

namespace whff {

// Edge-replicated 4x4 block (codec.py:157-164); a is row-major with pitch lda.
WHFF_HD void gather_block(const float* a, int64_t lda, int64_t rows, int64_t cols,
                          int64_t brow, int64_t bcol, float blk[16]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t r = brow * 4 + i;
    if (r > rows - 1) r = rows - 1;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t c = bcol * 4 + j;
      if (c > cols - 1) c = cols - 1;
      blk[4 * i + j] = ldg(a + r * lda + c);
    }
  }
}

// codec.py:186-190: code = frexp(max|x|).e + 160, 0 for an all-zero block
WHFF_HD uint32_t block_exponent(const float blk[16]) {
  float mx = 0.0f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float a = fabsf(blk[i]);
    mx = a > mx ? a : mx;
  }
  if (!(mx > 0.0f)) return 0;
  int e;
  frexp((double)mx, &e);
  return (uint32_t)(e + kEmaxBias);
}

WHFF_HD void fwd_lift(int64_t& x, int64_t& y, int64_t& z, int64_t& w) {  // codec.py:118-125
  x += w; x >>= 1; w -= x;
  z += y; z >>= 1; y -= z;
  x += z; x >>= 1; z -= x;
  w += y; w >>= 1; y -= w;
  w += y >> 1; y -= w >> 1;
}

// codec.py:193-198, :137-142, :239-243.  Returns false on coefficient overflow.
WHFF_HD bool block_coefficients(const float blk[16], uint32_t code, uint32_t mag[16],
                                uint32_t& negm) {
  negm = 0;
  if (code == 0) {
#pragma unroll
    for (int i = 0; i < 16; ++i) mag[i] = 0;
    return true;
  }
  const int emax = (int)code - kEmaxBias;
  const double scale = ldexp(1.0, kQuantBits - emax);
  int64_t t[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) t[i] = (int64_t)rint((double)blk[i] * scale);
#pragma unroll
  for (int i = 0; i < 4; ++i) fwd_lift(t[4 * i], t[4 * i + 1], t[4 * i + 2], t[4 * i + 3]);  // rows
#pragma unroll
  for (int i = 0; i < 4; ++i) fwd_lift(t[i], t[4 + i], t[8 + i], t[12 + i]);                  // columns
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const int64_t v = t[seq_pos(c)];
    const int64_t a = v < 0 ? -v : v;
    if (a >= ((int64_t)1 << kNPlanes)) ok = false;
    mag[c] = (uint32_t)a;
    if (v < 0) negm |= 1u << c;
  }
  return ok;
}

// codec.py:271-293 for one block: smallest plane count whose reconstruction is
// within tol at every valid position, or kNPlanes + 1 (raw escape).
WHFF_HD int select_planes(const float blk[16], uint32_t validm, uint32_t code,
                          const uint32_t mag[16], uint32_t negm, double tol) {
  for (int t = 0; t <= kNPlanes; ++t) {
    const uint32_t shift = (uint32_t)(kNPlanes - t);
    Decoded d;
#pragma unroll
    for (int c = 0; c < 16; ++c) d.mag[c] = shift >= 32 ? 0u : (mag[c] >> shift) << shift;
    d.negm = negm;
    d.emax = code;
    d.raw = 0;
    float dec[16];
    reconstruct_words(d, dec);
    double emx = 0.0;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (!((validm >> i) & 1u)) continue;
      const double e = fabs((double)dec[i] - (double)blk[i]);
      if (e != e) bad = true;
      emx = e > emx ? e : emx;
    }
    if (!bad && emx <= tol) return t;
  }
  return kNPlanes + 1;
}

// Bit sinks for _encode_one: count only, or emit big-endian bits into a
// payload (LE uint32 words) at an absolute bit offset with atomicOr at the
// two boundary words shared with neighbouring blocks.
struct CountSink {
  int n = 0;
  WHFF_HD void put(uint32_t) { ++n; }
};

struct WordSink {
  uint32_t* words;   // payload as LE uint32 words
  uint64_t pos;      // absolute bit position of the next bit
  uint32_t acc;      // big-endian accumulator for word (pos >> 5)
  int n;
  int limit;         // bits past the budget are dropped (K:266-270)
  WHFF_HD void put(uint32_t bit) {
    if (n >= limit) return;
    acc |= (bit & 1u) << (31 - (uint32_t)(pos & 31));
    ++pos;
    ++n;
    if ((pos & 31) == 0) {
      // flush the completed word (pos-1 is inside it)
      const uint64_t w = (pos - 1) >> 5;
      if (acc) {
#if defined(__CUDA_ARCH__)
        atomicOr(words + w, bswap32(acc));
#else
        words[w] |= bswap32(acc);
#endif
      }
      acc = 0;
    }
  }
  WHFF_HD void finish() {
    if ((pos & 31) != 0 && acc) {
#if defined(__CUDA_ARCH__)
      atomicOr(words + (pos >> 5), bswap32(acc));
#else
      words[pos >> 5] |= bswap32(acc);
#endif
    }
    acc = 0;
  }
};

// K:139-225.  Emits one block; returns the emitted length (pre budget pad).
template <typename Sink>
WHFF_HD int encode_one(const uint32_t mag[16], uint32_t negm, uint32_t code, int planes,
                       bool raw, const uint32_t raw_words[16], int budget,
                       bool has_raw_flag, Sink& out) {
  int n = 0;
  for (int i = 8; i >= 0; --i) { out.put((code >> i) & 1u); ++n; }
  if (has_raw_flag) { out.put(raw ? 1u : 0u); ++n; }
  if (raw) {
    for (int c = 0; c < 16; ++c)
      for (int i = 31; i >= 0; --i) { out.put((raw_words[c] >> i) & 1u); ++n; }
    return n;
  }
  if (code == 0) return n;
  uint32_t sig = 0;
  bool done = false;
  for (int p = kNPlanes - 1; p > kNPlanes - 1 - planes; --p) {
    if (done) break;
    for (int c = 0; c < 16; ++c) {                 // refinement pass
      if ((sig >> c) & 1u) {
        if (budget && n >= budget) { done = true; break; }
        out.put((mag[c] >> p) & 1u);
        ++n;
      }
    }
    if (done) break;
    uint32_t rem = ~sig & 0xFFFFu;                  // significance pass
    while (rem) {
      if (budget && n >= budget) { done = true; break; }
      uint32_t flag = 0;
      for (uint32_t r = rem; r; r &= r - 1) {
        const int c = (int)(31 - clz32(r & (0u - r)));
        if ((mag[c] >> p) & 1u) { flag = 1; break; }
      }
      out.put(flag);
      ++n;
      if (!flag) break;
      bool hit = false;
      for (uint32_t r = rem; r; r &= r - 1) {
        const uint32_t h = r & (0u - r);
        const int c = (int)(31 - clz32(h));
        if (budget && n >= budget) { done = true; break; }
        const uint32_t bit = (mag[c] >> p) & 1u;
        if (bit && budget && n == budget - 1) {     // sign would not fit
          out.put(0u);
          ++n;
          done = true;
          break;
        }
        out.put(bit);
        ++n;
        if (bit) {
          out.put((negm >> c) & 1u);
          ++n;
          sig |= h;
          rem = r & ~(h | (h - 1));                 // drop the consumed prefix
          hit = true;
          break;
        }
      }
      if (done || !hit) break;
    }
    if (done) break;
  }
  return n;
}

// Per-block plan shared by both encoder passes.
struct BlockPlan {
  uint32_t mag[16];
  uint32_t negm;
  uint32_t code;
  uint32_t raw_words[16];
  int planes;
  bool raw;
  bool ok;
};

// mode: 0 rate, 1 precision, 2 accuracy (codec.py:249-262)
WHFF_HD void plan_block(const float* a, int64_t lda, int64_t rows, int64_t cols,
                        int64_t b, int64_t bc, int mode, double param, BlockPlan& pl) {
  const int64_t brow = b / bc, bcol = b % bc;
  float blk[16];
  gather_block(a, lda, rows, cols, brow, bcol, blk);
  pl.code = block_exponent(blk);
  pl.ok = block_coefficients(blk, pl.code, pl.mag, pl.negm);
  pl.raw = false;
  pl.planes = kNPlanes;
  if (mode == 1) {
    const int p = (int)param;
    pl.planes = p < kNPlanes ? p : kNPlanes;
  } else if (mode == 2) {
    uint32_t validm = 0;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j)
        if (brow * 4 + i < rows && bcol * 4 + j < cols) validm |= 1u << (4 * i + j);
    int t = select_planes(blk, validm, pl.code, pl.mag, pl.negm, param);
    if (t > kNPlanes) { pl.raw = true; t = 0; }
    pl.planes = t;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    uint32_t u;
#if defined(__CUDA_ARCH__)
    u = __float_as_uint(blk[i]);
#else
    __builtin_memcpy(&u, &blk[i], 4);
#endif
    pl.raw_words[i] = pl.raw ? u : 0u;
  }
}

}  // namespace whff
