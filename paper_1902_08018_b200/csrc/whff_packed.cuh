// whff_packed.cuh -- the tile-packed device layout of a WHFZ stream and the
// fused decode + GEMV / decode-only kernels that read it.
//
// Why a second device layout.  The reference bitstream (codec.py:225-314,
// K:139-368) codes every 4x4 block as bit planes with group-tested
// significance: each block is a serial parse whose cost is ~1,000 thread
// instructions per 16-byte block on a B200, 11x the ~90 the
// SM can issue per block at HBM speed.  The information the GEMV needs per
// block is only (emax, 16 signed integer coefficients q_c) -- exactly what
// the reference's decode_blocks (K:371-408) hands to _reconstruct_blocks
// (codec.py:209-218).  At upload time this layout re-codes those values
// losslessly so that decoding is branch-free SIMT work:
//
//   band     = 4 block-rows (16 matrix rows)
//   tile     = band x 32 block-columns; lane l of a warp owns block-column
//              32 t + l of every block-row of the band
//   segment  = band x up to 8 tiles (256 block-columns) sharing one "field
//              profile": a width W_c per coefficient c (sequency order,
//              codec.py:40) = the widest value of c in the segment, and a
//              width W_e for emax - emax_base
//   record   = one block: [emax delta: W_e bits][field 0 .. field 15], the
//              fields at offsets fixed per segment; field 0 (DC) is two's
//              complement, fields 1..15 offset-binary (q + 2^(W-1)).
//
// Records are MSB-first bit strings of L bits (L per segment).  The 32
// records of one block-row of a tile form a "record group" of exactly L
// words: the first floor(L/32) words of each record interleaved across the
// lanes (word k of lane l at 32 k + l: one coalesced 128-byte load per k),
// then the 32 tails of L mod 32 bits packed back to back.  A tile is
// nrows record groups padded to 16 bytes; a segment body is its tiles.
//
// Fast path (every segment of a smooth WHFF operator, L <= 128): field c is
// read from a static register pair (a_k, a_k+1) of the record's four words,
// k = 0 for c <= 1, 0 or 1 for c = 2 (segment flag), 1 for c = 3..8 and 2
// for c = 9..15 (the packer pads so each field lies inside its pair), with
// two funnel shifts: the left one brings the field to the top, the right one
// shifts it down under the binary32 exponent of 2^23 ("magic number"), so
// float(2^23 + u) - (2^23 + 2^(W-1)) = q exactly (W <= 23).  Segments whose
// fields do not fit (adversarial data) take a generic per-lane path.
//
// Blocks the coefficient-domain evaluation cannot take (raw escapes, scales
// outside 2^-126..2^100; see coef_ok in whff_b200.cu) are "exceptions":
// their records are zero and their 16 decoded binary32 words (bit-exact
// with codec.decompress) live in a side list processed per segment.
//
// Everything the packer and the kernels share is __host__ __device__.
#pragma once

#include "whff_decode.cuh"

namespace whff {
namespace pk {

constexpr int kBand = 4;          // block-rows per band
constexpr int kTile = 32;         // block-columns per tile (one per lane)
constexpr int kSegTiles = 8;      // tiles per segment
constexpr int kSegCols = kTile * kSegTiles;
constexpr int kMagicW = 23;       // widest offset-binary field on the magic path
constexpr int kMaxRecordBits = 9 + 28 * 16;
constexpr int kMaxRecordWords = (kMaxRecordBits + 31) / 32;   // 15
constexpr uint32_t kMagic = 0x4B000000u;                      // binary32 2^23

// Segment header (48 bytes).
struct alignas(16) Seg {
  uint64_t body;       // word offset of the segment body
  uint32_t hdr;        // [0:9) emax_base [9:13) W_e [13] generic [14] k2 [16:25) L
  uint32_t w[3];       // W_c, 5 bits each: c = 6 * word + slot
  uint32_t o[4];       // fast path: offset of field c (7 bits): c = 4 * word + slot
  uint32_t exc_begin;  // first exception of the segment
  uint32_t exc_count;
};

WHFF_HD int seg_emax_base(const Seg& s) { return (int)(s.hdr & 511u); }
WHFF_HD int seg_We(const Seg& s) { return (int)((s.hdr >> 9) & 15u); }
WHFF_HD bool seg_generic(const Seg& s) { return (s.hdr >> 13) & 1u; }
WHFF_HD bool seg_k2(const Seg& s) { return (s.hdr >> 14) & 1u; }
WHFF_HD int seg_L(const Seg& s) { return (int)((s.hdr >> 16) & 511u); }
WHFF_HD int seg_W(const Seg& s, int c) { return (int)((s.w[c / 6] >> (5 * (c % 6))) & 31u); }
WHFF_HD int seg_o(const Seg& s, int c) { return (int)((s.o[c / 4] >> (8 * (c % 4))) & 127u); }

// static register pair of field c on the fast path (c = 2: the segment flag)
WHFF_HD int field_pair(int c, bool k2) { return c <= 1 ? 0 : c == 2 ? (k2 ? 1 : 0) : c <= 8 ? 1 : 2; }

// Field offsets from the widths (W[0] >= 1).  Fast layout: fields in order,
// each inside the 64-bit window of its static register pair (bits
// [32k, 32k + 64) of the record; padded up to 32k when needed); generic
// (fields back to back) when a field does not fit or a field c >= 1 is
// wider than the magic path allows.
struct Layout {
  int We, L;
  bool fast, k2;
  int o[16];
};
WHFF_HD void make_layout(int We, const int W[16], Layout& f) {
  int cur = We;
  bool fast = true, k2 = false;
  for (int c = 0; c < 16; ++c) {
    f.o[c] = 0;
    if (W[c] == 0) continue;
    int k;
    if (c <= 1) {
      k = 0;
    } else if (c == 2) {
      k = cur + W[c] <= 64 ? 0 : 1;
      k2 = k == 1;
    } else {
      k = c <= 8 ? 1 : 2;
    }
    if (c >= 3 && W[c] > kMagicW) fast = false;   // (c = 1, 2 convert as integers)
    if (cur < 32 * k) cur = 32 * k;
    if (cur + W[c] > 32 * k + 64) fast = false;
    f.o[c] = cur;
    cur += W[c];
  }
  if (!fast) {
    k2 = false;
    cur = We;
    for (int c = 0; c < 16; ++c) {
      f.o[c] = cur;
      cur += W[c];
    }
  }
  f.We = We;
  f.L = cur;
  f.fast = fast;
  f.k2 = k2;
}

// signed width: the fewest bits holding q in two's complement / offset binary
WHFF_HD int qwidth(int32_t q) {
  if (q == 0) return 0;
  const uint32_t a = (uint32_t)(q >= 0 ? q : ~q);
  return a == 0 ? 1 : 33 - (int)clz32(a);
}
WHFF_HD int bitwidth_u(uint32_t x) { return x == 0 ? 0 : 32 - (int)clz32(x); }

// words of one tile: nrows record groups of L words, padded to 16 bytes
WHFF_HD uint64_t tile_words(int nrows, int L) { return ((uint64_t)nrows * L + 3) & ~3ull; }

// Geometry of a packed stream.
struct Geom {
  uint64_t rows, cols, br, bc;
  uint64_t nband;   // ceil(br / 4)
  uint64_t ntile;   // tiles per band: ceil(bc / 32)
  uint64_t nsegb;   // segments per band: ceil(ntile / 8)
};
WHFF_HD Geom make_geom(uint64_t rows, uint64_t cols) {
  Geom g;
  g.rows = rows;
  g.cols = cols;
  g.br = (rows + 3) / 4;
  g.bc = (cols + 3) / 4;
  g.nband = (g.br + kBand - 1) / kBand;
  g.ntile = (g.bc + kTile - 1) / kTile;
  g.nsegb = (g.ntile + kSegTiles - 1) / kSegTiles;
  return g;
}
WHFF_HD int band_rows(const Geom& g, uint64_t band) {
  const uint64_t r = g.br - band * kBand;
  return r < (uint64_t)kBand ? (int)r : kBand;
}
WHFF_HD int seg_tiles(const Geom& g, uint64_t sb) {
  const uint64_t r = g.ntile - sb * kSegTiles;
  return r < (uint64_t)kSegTiles ? (int)r : kSegTiles;
}

// record bits: put the low W bits of val at record bits [pos, pos + W)
WHFF_HD void put_bits(uint32_t* rec, int pos, int W, uint32_t val) {
  if (W <= 0) return;
  const uint64_t v = (uint64_t)(val & (W >= 32 ? 0xFFFFFFFFu : ((1u << W) - 1u))) << (64 - W);
  const int w = pos >> 5, s = pos & 31;
  const uint64_t sh = v >> s;
  rec[w] |= (uint32_t)(sh >> 32);
  if (s + W > 32) rec[w + 1] |= (uint32_t)sh;
}
// W bits at record bits [pos, pos + W), W <= 32, unsigned
WHFF_HD uint32_t get_bits(const uint32_t* rec, int pos, int W) {
  if (W <= 0) return 0u;
  const int w = pos >> 5, s = pos & 31;
  const uint32_t hi = rec[w], lo = (s + W > 32) ? rec[w + 1] : 0u;
  const uint32_t x = fsl(hi, lo, (uint32_t)s);
  return W >= 32 ? x : x >> (32 - W);
}

// Record of one decoded block (q in sequency order) under a layout.
WHFF_HD void build_record(const Layout& f, const int W[16], uint32_t edelta, const int32_t q[16],
                          uint32_t* rec /* kMaxRecordWords, zeroed */) {
  put_bits(rec, 0, f.We, edelta);
  for (int c = 0; c < 16; ++c) {
    if (W[c] == 0) continue;
    const uint32_t u = c == 0 ? (uint32_t)q[c] : (uint32_t)(q[c] + (1 << (W[c] - 1)));
    put_bits(rec, f.o[c], W[c], u);
  }
}
// ...and its inverse (both paths: offsets from the layout)
WHFF_HD void parse_record(const Layout& f, const int W[16], const uint32_t* rec, uint32_t& edelta,
                          int32_t q[16]) {
  edelta = get_bits(rec, 0, f.We);
  for (int c = 0; c < 16; ++c) {
    if (W[c] == 0) {
      q[c] = 0;
      continue;
    }
    const uint32_t u = get_bits(rec, f.o[c], W[c]);
    if (c == 0) q[c] = (int32_t)(u << (32 - W[c])) >> (32 - W[c]);
    else q[c] = (int32_t)u - (1 << (W[c] - 1));
  }
}

// Coefficient-domain exceptions (codec.py:215-217 raw escapes; scales the
// binary32 sink cannot hold): identical to coef_ok() in whff_b200.cu.
WHFF_HD bool is_exception(const Decoded& d) {
  const int k = (int)d.emax - kEmaxBias - kQuantBits;
  return d.raw || (d.emax != 0 && !(k >= -126 && k <= 100));
}

WHFF_HD void signed_coefs(const Decoded& d, int32_t q[16]) {
  for (int c = 0; c < 16; ++c) {
    const int32_t m = (int32_t)d.mag[c];
    q[c] = ((d.negm >> c) & 1u) ? -m : m;
  }
}

// Words of a block from its signed coefficients (as reconstruct_words).
WHFF_HD void words_from_q(const int32_t q[16], uint32_t emax, float out[16]) {
  Decoded d;
  d.raw = 0;
  d.emax = emax;
  d.negm = 0;
  for (int c = 0; c < 16; ++c) {
    d.mag[c] = (uint32_t)(q[c] < 0 ? -q[c] : q[c]);
    if (q[c] < 0) d.negm |= 1u << c;
  }
  reconstruct_words(d, out);
}

// ---------------------------------------------------------------------------
// fast-path field extraction (shared by the kernels and the host check)
// ---------------------------------------------------------------------------
// Per-field parameters (a warp keeps them in shared memory):
// c = 0 (DC, two's complement): {W_e (left shift), 32 - W_0 (arithmetic
// right shift), -, -}.  c = 1, 2 (the large AC coefficients, up to 28 bits,
// converted as integers): {left shift inside the static pair (0..63), 0,
// 32 - W, 2^(W-1)}.  c >= 3 (W <= 23): {left shift, 2^23 >> W (high word of
// the magic right funnel), 32 - W (its shift), bits of -(2^23 + 2^(W-1))}.
// Absent fields give q = 0 on both paths.
struct alignas(16) FieldPar {
  uint32_t x, y, z, w;
};
WHFF_HD FieldPar field_param(const Seg& S, int c) {
  const int W = seg_W(S, c);
  FieldPar p;
  if (c == 0) {
    p.x = (uint32_t)seg_We(S);
    p.y = 32u - (uint32_t)W;
    p.z = 0u;
    p.w = 0u;
  } else if (W == 0) {
    p.x = 0u;
    p.y = c <= 2 ? 0u : kMagic;
    p.z = 32u;
    p.w = c <= 2 ? 0u : 0xCB000000u;         // -2^23
  } else {
    const int k = field_pair(c, seg_k2(S));
    p.x = (uint32_t)(seg_o(S, c) - 32 * k);
    p.y = c <= 2 ? 0u : kMagic >> W;
    p.z = 32u - (uint32_t)W;
    p.w = c <= 2 ? 1u << (W - 1) : 0xCB000000u + (1u << (W - 1));   // -(2^23 + 2^(W-1))
  }
  return p;
}

// high word of the 64-bit (hi:lo) << n, n in [0, 63]: one SHF.L.U64.HI
WHFF_HD uint32_t fsl64(uint32_t hi, uint32_t lo, uint32_t n) {
  return (uint32_t)(((((uint64_t)hi << 32) | lo) << n) >> 32);
}

// Field c >= 1 read from its register pair (hi, lo): the 64-bit left shift
// brings it to the top, the clamped right funnel shifts it under the
// exponent of 2^23, so the binary32 bits are 2^23 + u exactly; minus
// 2^23 + 2^(W-1) = q.
WHFF_HD float field_f(uint32_t hi, uint32_t lo, const FieldPar& p) {
  const uint32_t x = fsl64(hi, lo, p.x);
  const uint32_t fb = fsr(x, p.y, p.z);
#if defined(__CUDA_ARCH__)
  return __fadd_rn(__uint_as_float(fb), __uint_as_float(p.w));
#else
  return as_float(fb) + as_float(p.w);
#endif
}
WHFF_HD int32_t field_i(uint32_t hi, uint32_t lo, const FieldPar& p) {
  const uint32_t fb = fsr(fsl64(hi, lo, p.x), p.y, p.z);
  return (int32_t)(fb - (p.w & 0x7FFFFFFFu));
}
WHFF_HD int32_t field_dc(uint32_t a0, uint32_t a1, const FieldPar& p0) {
  return (int32_t)fsl64(a0, a1, p0.x) >> p0.y;
}
WHFF_HD uint32_t field_edelta(uint32_t a0, int We) { return fsr(a0, 0u, 32u - (uint32_t)We); }

// All 16 coefficients (sequency order) of one fast-path record a[0..3]
// (the host check's form; the kernels read par from shared memory).
WHFF_HD void fields_int(const uint32_t a[4], const FieldPar par[16], bool k2, int32_t q[16]) {
  q[0] = field_dc(a[0], a[1], par[0]);
  q[1] = field_i(a[0], a[1], par[1]);
  q[2] = k2 ? field_i(a[1], a[2], par[2]) : field_i(a[0], a[1], par[2]);
  for (int c = 3; c <= 8; ++c) q[c] = field_i(a[1], a[2], par[c]);
  for (int c = 9; c < 16; ++c) q[c] = field_i(a[2], a[3], par[c]);
}
}  // namespace pk
}  // namespace whff
static_assert(sizeof(whff::pk::Seg) == 48, "segment header is 48 bytes");
