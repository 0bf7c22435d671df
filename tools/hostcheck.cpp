// Host build of the device decoder (paper_1902_08018_b200/csrc/whff_decode.cuh)
// so its exact logic can be compared with the CPU oracle without a GPU.
// Built by tests/conftest.py into tools/libhostcheck.so (test-only).
#include <cstring>
#include "../paper_1902_08018_b200/csrc/whff_decode.cuh"

extern "C" {

// words: payload as little-endian uint32 words, zero padded (>= 8 words).
void hc_decode_blocks(const uint32_t* words, uint64_t payload_bits,
                      const uint64_t* offsets, const uint64_t* seglens,
                      int64_t nb, int planes_limit, int has_raw,
                      uint32_t* mag, uint8_t* neg, uint16_t* emax, uint8_t* raw,
                      uint32_t* raw_words, uint64_t* consumed) {
  for (int64_t b = 0; b < nb; ++b) {
    uint64_t start = offsets[b];
    uint64_t limit = start + seglens[b];
    if (limit > payload_bits) limit = payload_bits;
    int64_t len64 = (int64_t)limit - (int64_t)start;
    int len = len64 > 65535 ? 65535 : (int)len64;
    whff::BitWin bw;
    whff::win_at(bw, words, start, len);
    whff::Decoded d;
    // the kernels' dispatch: no refill when the segment fits the register
    const bool fits = whff::fits_no_refill(start, len);
    if (has_raw) {
      if (!fits) whff::decode_block<true, true>(bw, planes_limit, d, 1u);
      else whff::decode_block<true, false>(bw, planes_limit, d, 1u);
    } else {
      if (!fits) whff::decode_block<false, true>(bw, planes_limit, d, 1u);
      else whff::decode_block<false, false>(bw, planes_limit, d, 1u);
    }
    emax[b] = (uint16_t)d.emax;
    raw[b] = (uint8_t)d.raw;
    consumed[b] = (uint64_t)d.consumed;
    for (int c = 0; c < 16; ++c) {
      if (d.raw) {
        raw_words[16 * b + c] = d.mag[c];
        mag[16 * b + c] = 0;
      } else {
        mag[16 * b + c] = d.mag[c];
        raw_words[16 * b + c] = 0;
      }
      neg[16 * b + c] = (uint8_t)((d.negm >> c) & 1u);
    }
  }
}

// Full decode into a (rows, cols) float32 array (codec.decompress sans checks).
void hc_decompress(const uint32_t* words, uint64_t payload_bits,
                   const uint64_t* offsets, const uint64_t* seglens,
                   int64_t rows, int64_t cols, int planes_limit, int has_raw,
                   float* out) {
  int64_t bc = (cols + 3) / 4, br = (rows + 3) / 4;
  for (int64_t b = 0; b < br * bc; ++b) {
    uint64_t start = offsets[b];
    uint64_t limit = start + seglens[b];
    if (limit > payload_bits) limit = payload_bits;
    int64_t len64 = (int64_t)limit - (int64_t)start;
    int len = len64 > 65535 ? 65535 : (int)len64;
    whff::BitWin bw;
    whff::win_at(bw, words, start, len);
    whff::Decoded d;
    if (has_raw)   // always the refill path here, without the early exit
      whff::decode_block<true, true, false>(bw, planes_limit, d, 1u);
    else
      whff::decode_block<false, true, false>(bw, planes_limit, d, 1u);
    float blk[16];
    whff::reconstruct_words(d, blk);
    int64_t r0 = (b / bc) * 4, c0 = (b % bc) * 4;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j)
        if (r0 + i < rows && c0 + j < cols) out[(r0 + i) * cols + c0 + j] = blk[4 * i + j];
  }
}

}  // extern "C"

#include "../paper_1902_08018_b200/csrc/whff_encode.cuh"
extern "C" {
// Two-pass GPU-encoder logic on the host: returns total bits, fills offsets;
// when words != NULL also emits the payload (LE uint32 words, zeroed).
int64_t hc_compress(const float* a, int64_t rows, int64_t cols, int mode, double param,
                    uint64_t* offsets, uint32_t* words) {
  int64_t br = (rows + 3) / 4, bc = (cols + 3) / 4, nb = br * bc;
  int budget = mode == 0 ? (int)param * 16 : 0;
  bool has_raw = mode == 2;
  uint64_t total = 0;
  for (int64_t b = 0; b < nb; ++b) {
    whff::BlockPlan pl;
    whff::plan_block(a, cols, rows, cols, b, bc, mode, param, pl);
    if (!pl.ok) return -1;
    offsets[b] = total;
    int n;
    if (words) {
      whff::WordSink ws{words, total, 0u, 0, budget ? budget : 0x7FFFFFFF};
      n = whff::encode_one(pl.mag, pl.negm, pl.code, pl.planes, pl.raw, pl.raw_words,
                           budget, has_raw, ws);
      ws.finish();
    } else {
      whff::CountSink cs;
      n = whff::encode_one(pl.mag, pl.negm, pl.code, pl.planes, pl.raw, pl.raw_words,
                           budget, has_raw, cs);
    }
    if (budget) n = budget;
    total += (uint64_t)n;
  }
  return (int64_t)total;
}
}

extern "C" {
// K:228-283 encode_blocks from arrays with the device encoder logic.
int64_t hc_encode_blocks(const uint32_t* mag, const uint8_t* neg, const uint16_t* emax,
                         const uint8_t* planes, const uint8_t* raw_mask, const uint32_t* raw_words,
                         int64_t nb, int budget, int has_raw, uint64_t* offsets, uint32_t* words) {
  uint64_t total = 0;
  for (int64_t b = 0; b < nb; ++b) {
    uint32_t m[16], rw[16], negm = 0;
    for (int c = 0; c < 16; ++c) {
      m[c] = mag[16 * b + c];
      rw[c] = raw_words[16 * b + c];
      if (neg[16 * b + c]) negm |= 1u << c;
    }
    bool raw = has_raw && raw_mask[b];
    offsets[b] = total;
    int n;
    if (words) {
      whff::WordSink ws{words, total, 0u, 0, budget ? budget : 0x7FFFFFFF};
      n = whff::encode_one(m, negm, emax[b], planes[b], raw, rw, budget, has_raw != 0, ws);
      ws.finish();
    } else {
      whff::CountSink cs;
      n = whff::encode_one(m, negm, emax[b], planes[b], raw, rw, budget, has_raw != 0, cs);
    }
    if (budget) n = budget;
    total += (uint64_t)n;
  }
  return (int64_t)total;
}
}

#include "../paper_1902_08018_b200/csrc/whff_relayout.cuh"
extern "C" {
// forward / inverse skeleton-first permutation of every segment (out must
// start as a copy of in)
void hc_relayout(const uint32_t* in, uint32_t* out, const uint64_t* offsets, const uint64_t* seglens,
                 int64_t nb, uint64_t payload_bits, int planes_limit, int has_raw, int inverse) {
  for (int64_t b = 0; b < nb; ++b) {
    uint64_t start = offsets[b], limit = start + seglens[b];
    if (limit > payload_bits) limit = payload_bits;
    int64_t l = (int64_t)limit - (int64_t)start;
    int len = l > 65535 ? 65535 : (int)l;
    if (inverse) whff::unrelayout_segment(in, out, start, len, planes_limit, has_raw != 0);
    else whff::relayout_segment(in, out, start, len, planes_limit, has_raw != 0);
  }
}
// decode_blocks on a skeleton-first payload
void hc_decode_blocks_sf(const uint32_t* words, uint64_t payload_bits, const uint64_t* offsets,
                         const uint64_t* seglens, int64_t nb, int planes_limit, int has_raw,
                         uint32_t* mag, uint8_t* neg, uint16_t* emax, uint8_t* raw,
                         uint32_t* raw_words, uint64_t* consumed) {
  for (int64_t b = 0; b < nb; ++b) {
    uint64_t start = offsets[b], limit = start + seglens[b];
    if (limit > payload_bits) limit = payload_bits;
    int64_t l = (int64_t)limit - (int64_t)start;
    int len = l > 65535 ? 65535 : (int)l;
    whff::BitWin bw;
    whff::win_at(bw, words, start, len);
    whff::Decoded d;
    const bool fits = whff::fits_no_refill(start, len);
    if (has_raw) {
      if (!fits) whff::decode_block_sf<true, true>(bw, planes_limit, d);
      else whff::decode_block_sf<true, false>(bw, planes_limit, d);
    } else {
      if (!fits) whff::decode_block_sf<false, true>(bw, planes_limit, d);
      else whff::decode_block_sf<false, false>(bw, planes_limit, d);
    }
    emax[b] = (uint16_t)d.emax;
    raw[b] = (uint8_t)d.raw;
    consumed[b] = (uint64_t)d.consumed;
    for (int c = 0; c < 16; ++c) {
      mag[16 * b + c] = d.raw ? 0u : d.mag[c];
      raw_words[16 * b + c] = d.raw ? d.mag[c] : 0u;
      neg[16 * b + c] = (uint8_t)((d.negm >> c) & 1u);
    }
  }
}
}
extern "C" {
// walk statistics per block (skeleton-first payload): outer / hit iterations
void hc_walk_stats(const uint32_t* words, uint64_t payload_bits, const uint64_t* offsets,
                   const uint64_t* seglens, int64_t nb, int planes_limit, int has_raw,
                   int32_t* outer, int32_t* hits) {
  for (int64_t b = 0; b < nb; ++b) {
    uint64_t start = offsets[b], limit = start + seglens[b];
    if (limit > payload_bits) limit = payload_bits;
    int len = (int)(limit - start);
    whff::BitWin bw;
    whff::win_at(bw, words, start, len);
    int hb = has_raw ? 10 : 9;
    uint32_t code = bw.w0 >> 23;
    outer[b] = hits[b] = 0;
    if (code == 0 || (has_raw && ((bw.w0 >> 22) & 1u))) continue;
    whff::adv<true>(bw, hb);
    uint8_t psig[16];
    whff::SkelWalk<true> w(bw, psig);
    w.B = len - hb;
    w.run(planes_limit);
    outer[b] = w.iters;
    hits[b] = w.hit_iters + 1000 * w.fast_iters;
  }
}
}
