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

// ---------------------------------------------------------------------------
// Tile-packed layout (csrc/whff_packed.cuh): a host packer with the device
// packer's rules, and an unpacker that reads every fast-path record with
// the kernels' funnel/magic extraction and checks it against the generic
// parse.  The GPU tests compare the device packer's output with hc_pack.
// ---------------------------------------------------------------------------
#include <algorithm>
#include <vector>

#include "../paper_1902_08018_b200/csrc/whff_packed.cuh"

namespace {
struct HostStream {
  const uint32_t* mag;
  const uint8_t* neg;
  const uint16_t* emax;
  const uint8_t* raw;
  const uint32_t* raw_words;
};
whff::Decoded hs_block(const HostStream& h, uint64_t b) {
  whff::Decoded d;
  d.emax = h.emax[b];
  d.raw = h.raw[b];
  d.negm = 0;
  d.consumed = 0;
  for (int c = 0; c < 16; ++c) {
    d.mag[c] = d.raw ? h.raw_words[16 * b + c] : h.mag[16 * b + c];
    if (h.neg[16 * b + c]) d.negm |= 1u << c;
  }
  return d;
}
}  // namespace

extern "C" {

// Pack (mag, neg, emax, raw, raw_words) of a rows x cols stream of codec
// mode `mode` (0 rate, 1 precision, 2 accuracy: the segment size).  Pass NULL
// outputs to size: returns body words; *nseg_out, *nexc_out.
int64_t hc_pack(const uint32_t* mag, const uint8_t* neg, const uint16_t* emax, const uint8_t* raw,
                const uint32_t* raw_words, int64_t rows, int64_t cols, uint8_t* segs_out,
                uint32_t* body_out, uint64_t* exc_block_out, uint32_t* exc_words_out,
                int64_t* nseg_out, int64_t* nexc_out, int64_t* generic_out, int mode) {
  using namespace whff;
  const HostStream hs{mag, neg, emax, raw, raw_words};
  const pk::Geom g = pk::make_geom(rows, cols, pk::seg_tiles_for_mode(mode));
  const uint64_t nseg = g.nband * g.nsegb;
  uint64_t body = 0, nexc = 0, generic = 0;
  for (uint64_t sid = 0; sid < nseg; ++sid) {
    const uint64_t band = sid / g.nsegb, sb = sid % g.nsegb;
    const int nrows = pk::band_rows(g, band);
    const uint64_t col0 = sb * g.segt * pk::kTile, ncols = std::min<uint64_t>(g.segt * pk::kTile, g.bc - col0);
    int W[16] = {0};
    uint32_t emin = 0xFFFF, emx = 0, ne = 0;
    for (int i = 0; i < nrows; ++i)
      for (uint64_t c = 0; c < ncols; ++c) {
        const whff::Decoded d = hs_block(hs, (band * 4 + i) * g.bc + col0 + c);
        if (pk::is_exception(d)) { ++ne; continue; }
        if (d.emax == 0) continue;
        emin = std::min(emin, d.emax);
        emx = std::max(emx, d.emax);
        int32_t q[16];
        pk::signed_coefs(d, q);
        for (int k = 0; k < 16; ++k) W[k] = std::max(W[k], pk::qwidth(q[k]));
      }
    if (W[0] < 1) W[0] = 1;
    const uint32_t ebase = emx >= emin ? emin : 0u;
    const int We = emx > emin ? pk::bitwidth_u(emx - emin) : 0;
    pk::Layout f;
    pk::make_layout(We, W, f);
    if (!f.fast) ++generic;
    pk::Seg S;
    S.body = body;
    S.hdr = pk::seg_hdr(ebase, f);
    S.w[0] = S.w[1] = S.w[2] = 0;
    S.o[0] = S.o[1] = S.o[2] = S.o[3] = 0;
    for (int c = 0; c < 16; ++c) {
      S.w[c / 6] |= (uint32_t)W[c] << (5 * (c % 6));
      if (f.fast) S.o[c / 4] |= (uint32_t)f.o[c] << (8 * (c % 4));
    }
    S.exc_begin = (uint32_t)nexc;
    S.exc_count = ne;
    const int L = f.L, R = pk::rec_words(L);
    const uint64_t TW = pk::tile_words(L);
    const int ntl = pk::seg_tiles(g, sb);
    if (segs_out) std::memcpy(segs_out + 48 * sid, &S, 48);
    for (int tt = 0; tt < ntl; ++tt)
      for (int i = 0; i < nrows; ++i)
        for (int lane = 0; lane < 32; ++lane) {
          const uint64_t col = (sb * g.segt + tt) * pk::kTile + lane;
          const uint64_t b = (band * 4 + i) * g.bc + col;
          int32_t q[16] = {0};
          uint32_t ed = 0;
          bool isexc = false;
          whff::Decoded d;
          if (col < g.bc) {
            d = hs_block(hs, b);
            isexc = pk::is_exception(d);
            if (!isexc && d.emax != 0) {
              pk::signed_coefs(d, q);
              ed = d.emax - ebase;
            }
          }
          uint32_t rec[pk::kMaxRecordWords + 1] = {0};
          pk::build_record(f, W, ed, q, rec);
          if (body_out) {
            uint32_t* tp = body_out + body + tt * TW;
            for (int k = 0; k < R; ++k) tp[pk::tile_word(k, lane, i)] = rec[k];
          }
          if (isexc) {
            if (exc_block_out) {
              exc_block_out[nexc] = b;
              float x[16];
              whff::reconstruct_words(d, x);
              std::memcpy(exc_words_out + 16 * nexc, x, 64);
            }
            ++nexc;
          }
        }
    body += ntl * TW;
  }
  if (nseg_out) *nseg_out = (int64_t)nseg;
  if (nexc_out) *nexc_out = (int64_t)nexc;
  if (generic_out) *generic_out = (int64_t)generic;
  return (int64_t)body;
}

// Decode a packed stream to words; fast-path segments are read with the
// kernels' extraction (fields_int) and checked against parse_record.
// Returns the number of records where the two disagree.
int64_t hc_unpack(const uint8_t* segs_in, const uint32_t* body, const uint64_t* exc_block,
                  const uint32_t* exc_words, int64_t nexc, int64_t rows, int64_t cols, float* out, int mode) {
  using namespace whff;
  const pk::Geom g = pk::make_geom(rows, cols, pk::seg_tiles_for_mode(mode));
  int64_t bad = 0;
  for (uint64_t sid = 0; sid < g.nband * g.nsegb; ++sid) {
    pk::Seg S;
    std::memcpy(&S, segs_in + 48 * sid, 48);
    const uint64_t band = sid / g.nsegb, sb = sid % g.nsegb;
    const int nrows = pk::band_rows(g, band);
    int W[16];
    for (int c = 0; c < 16; ++c) W[c] = pk::seg_W(S, c);
    pk::Layout f;
    pk::make_layout(pk::seg_We(S), W, f);
    const int L = pk::seg_L(S), R = pk::rec_words(L);
    const uint64_t TW = pk::tile_words(L);
    pk::FieldPar par[16];
    for (int c = 0; c < 16; ++c) par[c] = pk::field_param(S, c);
    for (int tt = 0; tt < pk::seg_tiles(g, sb); ++tt)
      for (int i = 0; i < nrows; ++i)
        for (int lane = 0; lane < 32; ++lane) {
          const uint64_t col = (sb * g.segt + tt) * pk::kTile + lane;
          if (col >= g.bc) continue;
          const uint32_t* tp = body + S.body + tt * TW;
          uint32_t rec[pk::kMaxRecordWords + 1] = {0};
          for (int k = 0; k < R; ++k) rec[k] = tp[pk::tile_word(k, lane, i)];
          uint32_t ed;
          int32_t q[16];
          pk::parse_record(f, W, rec, ed, q);
          if (!pk::seg_generic(S)) {
            // the kernels' words: five registers (words past the record are 0)
            uint32_t a[pk::kFastWords] = {0, 0, 0, 0, 0};
            for (int k = 0; k < pk::kFastWords && k < R; ++k) a[k] = rec[k];
            int32_t qf[16];
            pk::fields_int(a, par, pk::seg_k2(S), pk::seg_kA(S), pk::seg_kB(S), qf);
            const uint32_t ef = pk::field_edelta(a[0], pk::seg_We(S));
            bool same = ef == ed;
            for (int c = 0; c < 16; ++c) same = same && qf[c] == q[c];
            // the magic-float values equal q exactly
            for (int c = 3; c < 16; ++c) {
              const int k = pk::field_pair(c, pk::seg_k2(S), pk::seg_kA(S), pk::seg_kB(S));
              same = same && pk::field_f(a[k], k + 1 < pk::kFastWords ? a[k + 1] : 0u, par[c]) == (float)q[c];
            }
            // c = 1, 2 in the magic-number format (seg_m12) give the same q
            if (pk::seg_m12(S))
              for (int c = 1; c <= 2; ++c) {
                const int k = pk::field_pair(c, pk::seg_k2(S), pk::seg_kA(S), pk::seg_kB(S));
                same = same && pk::field_f(a[k], a[k + 1], pk::seg_param(S, c)) == (float)q[c];
              }
            // the group path (k_pk_gemv2, groups of <= 23 bits) gives the same q
            for (int gg = 0; gg < 2; ++gg) {
              if (!pk::group_magic(S, gg)) continue;
              const int k = pk::field_pair(pk::group_first(gg), pk::seg_k2(S), pk::seg_kA(S), pk::seg_kB(S));
              const uint32_t x = pk::group_bits(a[k], k + 1 < pk::kFastWords ? a[k + 1] : 0u,
                                                pk::group_param(S, pk::group_first(gg)).w);
              for (int c = pk::group_first(gg); c <= pk::group_last(gg); ++c)
                same = same && pk::group_field_f(x, pk::group_param(S, c)) == (float)q[c];
            }
            if (!same) ++bad;
          }
          float x[16];
          pk::words_from_q(q, (uint32_t)pk::seg_emax_base(S) + ed, x);
          const uint64_t r0 = (band * 4 + i) * 4, c0 = col * 4;
          for (int rr = 0; rr < 4; ++rr)
            for (int j = 0; j < 4; ++j)
              if ((int64_t)(r0 + rr) < rows && (int64_t)(c0 + j) < cols) out[(r0 + rr) * cols + c0 + j] = x[4 * rr + j];
        }
  }
  for (int64_t e = 0; e < nexc; ++e) {
    const uint64_t b = exc_block[e];
    const uint64_t r0 = (b / g.bc) * 4, c0 = (b % g.bc) * 4;
    for (int k = 0; k < 16; ++k) {
      const uint64_t r = r0 + (k >> 2), c = c0 + (k & 3);
      if ((int64_t)r < rows && (int64_t)c < cols) std::memcpy(&out[r * cols + c], &exc_words[16 * e + k], 4);
    }
  }
  return bad;
}

}  // extern "C"
