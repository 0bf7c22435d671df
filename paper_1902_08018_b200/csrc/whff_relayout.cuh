// whff_relayout.cuh -- skeleton-first device layout of WHFZ blocks.
//
// The reference bitstream (K:139-225 / K:286-368) interleaves, plane by plane,
// the refinement bits of the significant coefficients with the significance
// pass ("skeleton": group flags, insignificant runs, hits, signs).  Decoding
// it on a SIMT machine costs ~2,000 instructions per block because every
// plane must be walked and refinement bits arrive in rank order (see
// whff_decode.cuh).  The skeleton-first layout is a lossless PERMUTATION of
// each block's segment, computed on the device at upload:
//
//     [header][skeleton bits, read order][refinement bits of coefficient 0,
//      plane order][... of coefficient 1]...[... of coefficient 15][tail]
//
// where "read order" and "tail" (the bits the reference decoder never reads)
// are defined by the reference parse itself.  Segment lengths, offsets, the
// index and the byte count are unchanged; the inverse permutation restores the
// reference bytes exactly (tests/test_relayout_host.py round-trips them).
//
// The decoder for this layout (decode_block_sf) reproduces the reference's
// outputs bit-exactly: it walks only the skeleton -- a run of quiet planes is
// a run of zero flag bits, skipped with one clz and budget arithmetic -- and
// then reads each coefficient's magnitude as one contiguous field.  No rank
// insertion, no PDEP and no bit-matrix transpose remain.
#pragma once
#include <stdint.h>
#include "whff_decode.cuh"

namespace whff {

// ---------------------------------------------------------------------------
// bit-serial exact parse that records the role of every bit read
// ---------------------------------------------------------------------------
struct RoleSink {
  uint32_t skel[48];     // skeleton bits, MSB-first
  int ns = 0;
  uint32_t ref[16];      // refinement bits per coefficient, MSB-first (<= 27 bits)
  int nref[16];
  WHFF_HD RoleSink() {
    for (int i = 0; i < 48; ++i) skel[i] = 0;
    for (int c = 0; c < 16; ++c) { ref[c] = 0; nref[c] = 0; }
  }
  WHFF_HD void skel_bit(uint32_t b) {
    if (b) skel[ns >> 5] |= 0x80000000u >> (ns & 31);
    ++ns;
  }
  WHFF_HD void ref_bit(int c, uint32_t b) {
    ref[c] = (ref[c] << 1) | b;
    ++nref[c];
  }
};

// single-bit reader over a segment (positions relative to its start)
struct SegBits {
  const uint32_t* words;  // LE payload words
  uint64_t start;
  int len;
  WHFF_HD uint32_t get(int pos) const {
    const uint64_t a = start + (uint64_t)pos;
    return (bswap32(ldg(words + (a >> 5))) >> (31 - (a & 31))) & 1u;
  }
};

// K:286-368 with role recording.  Returns the bits consumed and whether the
// block has a permutable plane section (not raw / zero / truncated header).
WHFF_HD int parse_roles(const SegBits& in, int planes_limit, bool has_raw, RoleSink& rs,
                        int& hdr_bits, bool& permutable) {
  int pos = 0;
  const int limit = in.len;
  permutable = false;
  hdr_bits = 0;
  int code = 0;
  for (int i = 0; i < 9; ++i) {
    if (pos >= limit) return pos;
    code = (code << 1) | (int)in.get(pos++);
  }
  if (has_raw) {
    if (pos >= limit) return pos;
    if (in.get(pos++)) {                     // raw escape: 16 verbatim words
      const int end = pos + 512;
      return end < limit ? end : limit;
    }
  }
  if (code == 0) return pos;
  hdr_bits = pos;
  permutable = true;
  uint32_t sig = 0;
  const int pl = planes_limit < kNPlanes ? planes_limit : kNPlanes;
  for (int t = 0; t < pl; ++t) {
    const int p = 26 - t;
    (void)p;
    if (pos >= limit) break;
    for (int c = 0; c < 16; ++c) {           // refinement pass
      if ((sig >> c) & 1u) {
        if (pos >= limit) return pos;
        rs.ref_bit(c, in.get(pos++));
      }
    }
    uint32_t rem = ~sig & 0xFFFFu;           // significance pass
    while (rem) {
      if (pos >= limit) return pos;
      const uint32_t flag = in.get(pos++);
      rs.skel_bit(flag);
      if (!flag) break;
      bool hit = false;
      for (uint32_t r = rem; r; r &= r - 1) {
        const uint32_t h = r & (0u - r);
        if (pos >= limit) return pos;
        const uint32_t v = in.get(pos++);
        rs.skel_bit(v);
        if (v) {
          if (pos >= limit) return pos;      // sign unavailable
          rs.skel_bit(in.get(pos++));
          sig |= h;
          rem = r & ~(h | (h - 1));
          hit = true;
          break;
        }
      }
      if (!hit) break;
    }
  }
  return pos;
}

// bit writer into a local word buffer (MSB-first)
WHFF_HD void put_bits(uint32_t* o, int& at, uint32_t v, int n) {  // n <= 32, v in low n bits
  if (n <= 0) return;
  v = n == 32 ? v : (v & ((1u << n) - 1u));
  const int w = at >> 5, off = at & 31;
  const int room = 32 - off;
  if (n <= room) {
    o[w] |= v << (room - n);
  } else {
    o[w] |= v >> (n - room);
    o[w + 1] |= v << (32 - (n - room));
  }
  at += n;
}

// Replace segment bits [0, nbits) of the output payload with the first nbits
// of `o` (MSB-first).  Neighbouring blocks share boundary words, so the
// update is two atomic bitwise ops on disjoint bits.
WHFF_HD void store_bits(uint32_t* out_words, uint64_t start, const uint32_t* o, int nbits) {
  for (int i = 0; i < nbits;) {
    const uint64_t a = start + (uint64_t)i;
    const int off = (int)(a & 31);
    const int take = (32 - off) < (nbits - i) ? (32 - off) : (nbits - i);
    // bits [i, i+take) of o, aligned to word offset `off`
    const int w = i >> 5, s = i & 31;
    uint32_t chunk = (o[w] << s) | (s ? (o[w + 1] >> (32 - s)) : 0u);   // o bits from i, MSB-first
    chunk = take == 32 ? chunk : (chunk & ~(0xFFFFFFFFu >> take));      // keep `take` bits
    const uint32_t be = chunk >> off;                                   // into word position
    const uint32_t mask = (take == 32 ? 0xFFFFFFFFu : ~(0xFFFFFFFFu >> take)) >> off;
    uint32_t* dst = out_words + (a >> 5);
#if defined(__CUDA_ARCH__)
    atomicAnd(dst, ~bswap32(mask));
    atomicOr(dst, bswap32(be));
#else
    *dst = (*dst & ~bswap32(mask)) | bswap32(be);
#endif
    i += take;
  }
}

// Forward permutation of one block segment (out_words must hold a copy of the
// input payload: the tail and any gaps stay as they are).
WHFF_HD void relayout_segment(const uint32_t* in_words, uint32_t* out_words, uint64_t start,
                              int len, int planes_limit, bool has_raw) {
  SegBits in{in_words, start, len};
  RoleSink rs;
  int hdr = 0;
  bool perm = false;
  const int consumed = parse_roles(in, planes_limit, has_raw, rs, hdr, perm);
  if (!perm) return;                         // raw / zero / truncated: verbatim
  uint32_t o[48];
  for (int i = 0; i < 48; ++i) o[i] = 0;
  int at = 0;
  for (int i = 0; i < hdr; ++i) put_bits(o, at, in.get(i), 1);
  for (int i = 0; i < rs.ns; ++i) put_bits(o, at, (rs.skel[i >> 5] >> (31 - (i & 31))) & 1u, 1);
  for (int c = 0; c < 16; ++c) put_bits(o, at, rs.ref[c], rs.nref[c]);
  (void)consumed;
  store_bits(out_words, start, o, at);
}

// ---------------------------------------------------------------------------
// Skeleton-first decoder
// ---------------------------------------------------------------------------
// Skeleton walk with the reference's bit budget B (= segment bits after the
// header): refinement of plane P costs n bits, its significance pass costs
// the skeleton bits it reads.  Runs of quiet planes (flag 0) are skipped in
// bulk.  Outputs per coefficient the plane at which it became significant
// (psig, local memory), and (p_last, cut, sig_last): the last plane whose
// refinement was read, how many of its ranks got a bit, and the significant
// set at that refinement.
#ifndef WHFF_WALK_FAST
#define WHFF_WALK_FAST 1
#endif
template <bool REFILL>
struct SkelWalk {
  BitWin& bw;
  uint8_t* psig;
  uint32_t sig = 0;     // significant set; signs live in bit 7 of the psig bytes
  int n = 0;
  int B = 0;
  int t = 0;           // current plane index from the top (P = 26 - t)
  int p_last = 26, cut = 0;
  uint32_t sig_last = 0;
  uint32_t rem_lo = 0xFFFFu;   // coefficients still eligible in plane t (above its last hit)
  bool ended = false;
  WHFF_HD SkelWalk(BitWin& b, uint8_t* ps) : bw(b), psig(ps) {}

  // refinement of the plane at index t
  WHFF_HD void refine() {
    p_last = 26 - t;
    sig_last = sig;
    rem_lo = 0xFFFFu;
    if (B < n) { cut = B; B = 0; ended = true; return; }
    B -= n;
    cut = n;
  }
  // advance to the next plane (and read its refinement) or end
  WHFF_HD void next_plane(int pl) {
    if (t + 1 >= pl) { ended = true; return; }
    ++t;
    refine();
  }

  int iters = 0, hit_iters = 0, fast_iters = 0;   // instrumentation (host statistics)
  WHFF_HD void run(int pl) {
    t = 0;
    refine();                                // plane 26: n = 0
#if WHFF_WALK_FAST
    run_fast(pl);
#endif
    run_from(pl);
  }

  // Event loop.  One iteration consumes one token of the skeleton,
  //   0^m 1 0^z 1 s
  // = m zero group flags (each ends a plane; the next plane's refinement
  // costs n bits of budget), a raised flag, z insignificant coefficients of
  // the remainder, the hit and its sign.  The insignificant coefficients are
  // kept as an ordered nibble list, so the hit is nibble (off + z) and
  // removing it is a masked 64-bit merge (no per-coefficient loop).  A token
  // that would cross the budget, the plane limit or the window, or that has
  // no hit, leaves the loop untouched; the closed-form ending below resolves
  // the usual cases, and run_from() finishes any other block with the
  // general (reference-order) logic from exactly this state.
  WHFF_HD void run_fast(int pl) {
    if (ended) return;
    uint64_t ins = 0xFEDCBA9876543210ull;    // insignificant coefficients, nibble i = i-th
    int cnt = 16, off = 0;
    int P = 26 - t;                          // current plane
    const int Pmin = 27 - pl;                // planes P >= Pmin exist (t < pl)
    int nn = n, BB = B;
    uint32_t sg = sig, sl = sig_last;
    int aa = 0;      // the last hit emptied the remainder: plane P ends without a flag
    while (true) {
      const uint32_t x = bw.w0;
      const uint32_t m0 = clz_sh(x);         // zero flags (0xFFFFFFFF if x == 0)
      const uint32_t y = fsl(x, 0u, m0 + 1u);
      const uint32_t z = clz_sh(y);          // run before the hit (0xFFFFFFFF: none in w0)
      const int m = (int)m0 + aa;            // planes ended by this token
      const int base = m ? 0 : off;
      const int cost = (int)m0 * (nn + 1) + aa * nn + (int)z + 3;
      // fast iff: a hit among the remainder, the token inside w0 (m0 + z + 3
      // <= 32), every crossed plane exists and the budget covers the token
      const int chk = (29 - (int)m0 - (int)z) | (P - m - Pmin) | (BB - cost);
      if (!(z < (uint32_t)(cnt - base) && chk >= 0)) break;
#if !defined(__CUDA_ARCH__)
      ++fast_iters;
#endif
      const uint32_t sgn7 = (y >> (23u - z)) & 0x80u;   // the sign, at bit 7
      adv<REFILL>(bw, m0 + z + 3u);
      BB -= cost;
      P -= m;
      if (m) sl = sg;                        // sig at the refinement of plane P
      const int a = base + (int)z;
      const uint32_t c = (uint32_t)(ins >> (4 * a)) & 15u;
      const uint64_t lowm = (1ull << (4 * a)) - 1ull;
      ins = (ins & lowm) | ((ins >> 4) & ~lowm);
      cnt -= 1;
      psig[c] = (uint8_t)(P | sgn7);
      sg |= 1u << c;
      nn += 1;
      off = a;
      aa = a == cnt;
    }
    // Closed-form ending.  From the loop's exit state the reference reads on
    // until the budget or the plane limit stops it; when no further hit can
    // become significant the result is (p_last, cut, sig_last, flag bits
    // read) in closed form:
    //  * a pending implicit plane end (aa) charges the next plane's refinement;
    //  * the budget runs out inside the next run of zero flags: q complete
    //    (flag + n-bit refinement) pairs, then r < n+1 bits = a zero flag and
    //    r-1 refinement bits (or the flag that ends the last plane);
    //  * or inside the next event token 0^m0 1 0^z 1 s: its m0 quiet planes are
    //    complete and the hit or its sign is out of budget, so nothing changes.
    // Anything else (all significant, a flag without a hit, a token beyond the
    // window, plane limit inside a token) is run_from's.
    if (nn < 16) {
      int Pc = P, Bc = BB;
      uint32_t slc = sl;
      int offc = off;
      bool done = false;
      int pl_ = P, ct = 0, f = 0;
      uint32_t sl_ = sl;
      if (aa) {                              // implicit end of plane P (no flag)
        if (Pc - 1 < Pmin) { done = true; pl_ = Pc; sl_ = slc; ct = (int)popc32(slc); }
        else if (Bc < nn) { done = true; pl_ = Pc - 1; sl_ = sg; ct = Bc; }
        else { Pc -= 1; Bc -= nn; slc = sg; offc = 0; }
      }
      if (!done) {
        const uint32_t x = bw.w0;
        const uint32_t zf = clz_sh(x);
        const int m0 = zf > 32u ? 32 : (int)zf;    // zero flags available
        const int per = nn + 1;
        const int Q = Pc - Pmin;             // planes left below Pc
        const int q = small_div(Bc, per);
        const int r = Bc - q * per;
        int need;                            // zero flags the closed form reads
        if (q <= Q) {                        // the budget ends first
          f = q + (r > 0);
          need = f;
          if (f <= m0) {
            done = true;
            if (r > 0 && q == Q) {           // that flag ends the last plane
              pl_ = Pc - q; sl_ = q ? sg : slc; ct = q ? nn : (int)popc32(slc);
            } else if (f == 0) {
              pl_ = Pc; sl_ = slc; ct = (int)popc32(slc);
            } else {
              pl_ = Pc - f; sl_ = sg; ct = r > 0 ? r - 1 : nn;
            }
          }
        } else {                             // the planes end first (budget to spare)
          need = Q + 1;
          if (Q + 1 <= m0) {
            done = true;
            f = Q + 1;
            pl_ = Pc - Q; sl_ = Q ? sg : slc; ct = Q ? nn : (int)popc32(slc);
          }
        }
        if (!done && m0 < need && m0 <= Q) {   // an event token comes first
          const uint32_t y = fsl(x, 0u, (uint32_t)m0 + 1u);
          const int z = (int)clz32(y);
          const int krem = cnt - (m0 ? 0 : offc);
          const int b2 = Bc - m0 * per;
          if (z < krem && b2 < z + 3 && m0 + z + 3 <= 32) {
            done = true;
            f = m0 + (b2 < z + 2 ? b2 : z + 2);
            pl_ = Pc - m0; sl_ = m0 ? sg : slc; ct = m0 ? nn : (int)popc32(slc);
          }
        }
      }
      if (done) {
        adv<REFILL>(bw, (uint32_t)f);
        n = nn; sig = sg; B = 0;
        sig_last = sl_; p_last = pl_; cut = ct; t = 26 - pl_;
        ended = true;
        return;
      }
    }
    t = 26 - P; n = nn; B = BB; sig = sg;
    sig_last = sl;
    p_last = P;
    cut = (int)popc32(sl);
    // eligible remainder of plane t = ins[off:], i.e. every coefficient from
    // ins[off] up (all lower ones are significant or already skipped); empty
    // when the last hit took the remainder's last member (run_from ends the plane)
    rem_lo = off == 0 ? 0xFFFFu
           : off >= cnt ? 0u : (0xFFFFu << (uint32_t)((ins >> (4 * off)) & 15u)) & 0xFFFFu;
  }

  // general walk from any state "refinement of plane t read, next read is a
  // group flag of plane t (or the plane is exhausted)"
  WHFF_HD void run_from(int pl) {
    while (!ended) {
#if !defined(__CUDA_ARCH__)
      ++iters;
#endif
      const uint32_t remv = ~sig & rem_lo & 0xFFFFu;
      if (remv == 0) {                       // remainder empty: no flag, plane ends
        if (n == 16 && rem_lo == 0xFFFFu) {  // all significant: whole refinement planes
          int m = pl - 1 - t;
          if (m * 16 > B) m = B >> 4;
          if (m > 0) {
            t += m;
            B -= m * 16;
            p_last = 26 - t;
            sig_last = sig;
            cut = 16;
          }
        }
        next_plane(pl);
        continue;
      }
      // bulk: m quiet planes = m zero flags + (m) next refinements of n bits
      {
        const int zf = (int)clz32(bw.w0);
        int m = zf;
        const int planes_left = pl - 1 - t;
        if (m > planes_left) m = planes_left;
        if (m * (n + 1) > B) m = small_div(B, n + 1);    // budget boundary (once per block)
        if (m > 0) {
          adv<REFILL>(bw, (uint32_t)m);
          B -= m * (n + 1);
          t += m;
          p_last = 26 - t;
          sig_last = sig;
          cut = n;
          rem_lo = 0xFFFFu;
          continue;
        }
      }
      // one plane's flag at the boundary of budget / planes / window
      if (B == 0) { ended = true; break; }
      const uint32_t flag = bw.w0 >> 31;
      adv<REFILL>(bw, 1);
      B -= 1;
      if (!flag) { next_plane(pl); continue; }
      events(pl);
    }
  }

  // significance events of plane P = 26 - t after a raised flag
  WHFF_HD void events(int pl) {
    const int P = 26 - t;
    uint32_t rem = ~sig & rem_lo & 0xFFFFu;
    int krem = (int)popc32(rem);
    while (true) {
#if !defined(__CUDA_ARCH__)
      ++hit_iters;
#endif
      const uint32_t y = bw.w0;
      const int z = (int)clz32(y);
      if (z >= krem) {                       // no hit: krem zeros
        if (B < krem) {                      // the reference read B of them
          adv<REFILL>(bw, (uint32_t)B);
          B = 0;
          ended = true;
          return;
        }
        adv<REFILL>(bw, (uint32_t)krem);
        B -= krem;
        break;
      }
      if (B < z + 1) {                       // run or hit past the budget:
        adv<REFILL>(bw, (uint32_t)B);        // B zeros of the run were read
        B = 0;
        ended = true;
        return;
      }
      if (B == z + 1) {                          // sign unavailable (K:353-354)
        adv<REFILL>(bw, (uint32_t)(z + 1));
        B = 0;
        ended = true;
        return;
      }
      const uint32_t sgn = (y << (z + 1)) >> 31;
      B -= z + 2;
      for (int i = 0; i < z; ++i) rem &= rem - 1;
      const uint32_t h = rem & (0u - rem);
      rem ^= h;
      krem -= z + 1;
      psig[31 - clz32(h)] = (uint8_t)(P | (sgn << 7));
      sig |= h;
      n += 1;
      rem_lo = 0xFFFFu & ~(h | (h - 1u));
      if (krem == 0 || B == 0) {             // no further flag (remainder empty / budget)
        adv<REFILL>(bw, (uint32_t)(z + 2));
        if (krem != 0) { ended = true; return; }
        break;
      }
      // next group flag sits right after the sign (z + 3 <= 18 bits into y)
      const uint32_t f = (y << (z + 2)) >> 31;
      adv<REFILL>(bw, (uint32_t)(z + 3));
      B -= 1;
      if (!f) break;
    }
    next_plane(pl);
  }
};

// Per-coefficient consumer of the fields loop (the fused GEMV's coefficient-
// domain accumulator plugs in here); the default does nothing.
struct NullSink {
  template <int C>
  WHFF_HD void coef(uint32_t, uint32_t) {}
};

// MAGS = false: only the sink sees the magnitudes (d.mag is left unset, and
// so are raw-escape words: the caller re-decodes such blocks with MAGS).
// GROUPED: the fields loop leaves the coefficient chain once no lane has
// higher coefficients (a win for sparse blocks: accuracy / precision modes;
// FixedRate(8) blocks are dense enough that the extra branches cost ~0.5 %).
template <bool HAS_RAW, bool REFILL, class Sink = NullSink, bool MAGS = true, bool GROUPED = true>
WHFF_HD void decode_block_sf(BitWin& bw, int planes_limit, Decoded& d, Sink&& sink = Sink()) {
  const int len = bw.len;
  d.negm = 0;
  d.emax = 0;
  d.raw = 0;
  if (MAGS) {
#pragma unroll
    for (int c = 0; c < 16; ++c) d.mag[c] = 0;
  }
  if (len < 9) { d.consumed = len < 0 ? 0 : len; return; }
  const uint32_t hdr = bw.w0;
  const uint32_t code = hdr >> 23;
  d.emax = code;
  int hbits = 9;
  if (HAS_RAW) {
    if (len < 10) { d.consumed = 9; return; }
    if ((hdr >> 22) & 1u) {                  // raw escape: same as WHFZ
      adv<REFILL>(bw, 10);
      d.raw = 1;
      if (!MAGS) return;
      int nw = (len - 10) >> 5;
      if (nw > 16) nw = 16;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        if (c < nw) {
          d.mag[c] = bw.w0;
          adv<REFILL>(bw, 32);
        }
      }
      d.consumed = (len - 10 >= 512) ? 522 : len;
      return;
    }
    hbits = 10;
  }
  adv<REFILL>(bw, (uint32_t)hbits);
  if (code == 0) { d.consumed = hbits; return; }

  const int pl = planes_limit < kNPlanes ? planes_limit : kNPlanes;
  if (pl <= 0) { d.consumed = hbits; return; }
  alignas(16) uint32_t psw[4] = {0u, 0u, 0u, 0u};   // psig bytes (0 for insignificant)
  SkelWalk<REFILL> w(bw, reinterpret_cast<uint8_t*>(psw));
  w.B = len - hbits;
  w.run(pl);
  // Coefficient-major refinement fields, index order (K:326-332 bits).
  // Coefficient c, significant at plane ps, holds the bits of planes
  // ps-1 .. e: e = p_last+1 for the members of sig_last (one lower for the
  // first `cut` of them, which got plane p_last's bit), e = ps otherwise.
  // Its magnitude is the leading 1 at bit ps followed by the l = ps - e field
  // bits: funnelshift_r(F, 1, 32 - l) << e.
  const uint32_t sig = w.sig, sig_last = w.sig_last;
  const uint32_t pl1 = (uint32_t)(w.p_last + 1);
  const int cut = w.cut;
  int rank = 0;                              // running rank within sig_last
  uint32_t pv[4];
#if defined(__CUDA_ARCH__)
  {
    const uint4 q = *reinterpret_cast<const uint4*>(psw);    // one LDL.128
    pv[0] = q.x; pv[1] = q.y; pv[2] = q.z; pv[3] = q.w;
  }
#else
  for (int i = 0; i < 4; ++i) pv[i] = psw[i];
#endif
  unroll16_live<0, GROUPED>(sig, [&](auto cc) {
    constexpr int c = decltype(cc)::value;
    if ((sig >> c) & 1u) {                   // skipped when no lane of the warp has it
      const uint32_t pb = pv[c >> 2] >> (8 * (c & 3));
      const uint32_t ps = pb & 0x1Fu;
      uint32_t e = ps;
      if ((sig_last >> c) & 1u) {
        e = pl1 - (rank < cut ? 1u : 0u);
        ++rank;
      }
      const uint32_t l = ps - e;             // field length
      const uint32_t mag = fsr(bw.w0, 1u, 32u - l) << e;   // (1 : top l bits of F) << e
      if (MAGS) d.mag[c] = mag;
      sink.template coef<c>(mag, pb << 24);  // sign at bit 31
      adv<REFILL>(bw, l);
    }
  });
  if (MAGS) {                                // signs: bit 7 of each psig byte
    uint32_t nm = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) nm |= (((pv[i] & 0x80808080u) * 0x00204081u) >> 28) << (4 * i);
    d.negm = nm;
  }
  d.consumed = bw.pos;
}

// ---------------------------------------------------------------------------
// Inverse permutation (skeleton-first -> reference bytes)
// ---------------------------------------------------------------------------
// Pass 1 walks the skeleton to learn every coefficient's refinement length;
// pass 2 replays the reference's read order, drawing skeleton bits and each
// coefficient's refinement bits from their regions.
WHFF_HD void unrelayout_segment(const uint32_t* in_words, uint32_t* out_words, uint64_t start,
                                int len, int planes_limit, bool has_raw) {
  SegBits in{in_words, start, len};
  if (len < 9) return;
  int code = 0;
  for (int i = 0; i < 9; ++i) code = (code << 1) | (int)in.get(i);
  int hbits = 9;
  if (has_raw) {
    if (len < 10) return;
    if (in.get(9)) return;                   // raw: verbatim
    hbits = 10;
  }
  if (code == 0) return;
  // pass 1: the decoder's skeleton walk on the permuted segment
  BitWin bw;
  win_at(bw, in_words, start, len);
  adv<true>(bw, (uint32_t)hbits);
  const int pl = planes_limit < kNPlanes ? planes_limit : kNPlanes;
  if (pl <= 0) return;
  uint8_t psig[16];
  SkelWalk<true> w(bw, psig);
  w.B = len - hbits;
  w.run(pl);
  const int skel_end = bw.pos;                // end of the skeleton region
  int rstart[16], rlen[16];
  int at = skel_end;
  for (int c = 0; c < 16; ++c) {
    int l = 0;
    if ((w.sig >> c) & 1u) {
      l = (psig[c] & 0x1F) - 1 - w.p_last;   // bit 7 holds the sign
      l = l < 0 ? 0 : l;
      if ((w.sig_last >> c) & 1u) {
        const int rank = (int)popc32(w.sig_last & ((1u << c) - 1u));
        l += rank < w.cut ? 1 : 0;
      }
    }
    rstart[c] = at;
    rlen[c] = l;
    at += l;
  }
  // pass 2: replay K:286-368 order
  uint32_t o[48];
  for (int i = 0; i < 48; ++i) o[i] = 0;
  int wr = 0;
  for (int i = 0; i < hbits; ++i) put_bits(o, wr, in.get(i), 1);
  int sk = hbits;                             // skeleton cursor
  int rc[16];
  for (int c = 0; c < 16; ++c) rc[c] = 0;
  int pos = hbits;                            // reference read position
  const int limit = len;
  uint32_t sig = 0;
  bool stop = false;
  for (int t = 0; t < pl && !stop; ++t) {
    if (pos >= limit) break;
    for (int c = 0; c < 16 && !stop; ++c) {
      if ((sig >> c) & 1u) {
        if (pos >= limit) { stop = true; break; }
        const uint32_t b = rc[c] < rlen[c] ? in.get(rstart[c] + rc[c]) : 0u;
        ++rc[c];
        put_bits(o, wr, b, 1);
        ++pos;
      }
    }
    if (stop) break;
    uint32_t rem = ~sig & 0xFFFFu;
    while (rem && !stop) {
      if (pos >= limit) { stop = true; break; }
      const uint32_t flag = in.get(sk++);
      put_bits(o, wr, flag, 1);
      ++pos;
      if (!flag) break;
      bool hit = false;
      for (uint32_t r = rem; r; r &= r - 1) {
        const uint32_t h = r & (0u - r);
        if (pos >= limit) { stop = true; break; }
        const uint32_t v = in.get(sk++);
        put_bits(o, wr, v, 1);
        ++pos;
        if (v) {
          if (pos >= limit) { stop = true; break; }
          put_bits(o, wr, in.get(sk++), 1);
          ++pos;
          sig |= h;
          rem = r & ~(h | (h - 1));
          hit = true;
          break;
        }
      }
      if (!hit) break;
    }
  }
  store_bits(out_words, start, o, wr);
}

}  // namespace whff
