// whff_pack.cu -- the packer: a WHFZ stream on the device (reference or
// skeleton-first layout, any index) -> the tile-packed layout of
// whff_packed.cuh.  Two passes over the stream with the general block
// decoder (the same decode_any the decode-only kernels use): pass 1 sizes
// every segment, pass 2 writes the records and the exception side list.
#include <type_traits>

#include "whff_common.cuh"
#include "whff_packed.cuh"
#include "whff_packed_api.h"

static unsigned grid_of(uint64_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }

// ---------------------------------------------------------------------------
// packer, pass 1: per segment widths, emax range, exceptions, size
// ---------------------------------------------------------------------------
// One warp per segment; lane-strided over the segment's blocks, each decoded
// from the source stream with the general decoder (any layout, any index).
template <bool HAS_RAW>
#ifndef WHFF_PK_MINB
#define WHFF_PK_MINB 1
#endif
__global__ void __launch_bounds__(256, WHFF_PK_MINB) k_pk_stats(StreamView s, pk::Geom g, pk::Seg* segs,
                                                  uint64_t* seg_words, uint64_t* seg_exc) {
  const uint64_t sid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (sid >= g.nband * g.nsegb) return;
  const uint64_t band = sid / g.nsegb, sb = sid % g.nsegb;
  const int nrows = pk::band_rows(g, band);
  const uint64_t col0 = sb * g.segt * pk::kTile;
  const uint64_t ncols = min(g.segt * pk::kTile, g.bc - col0);
  uint32_t wmax[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) wmax[c] = 0;
  uint32_t emin = 0xFFFFu, emx = 0, nexc = 0;
  const uint64_t n = (uint64_t)nrows * ncols;
  for (uint64_t idx = lane; idx < n; idx += 32) {
    const uint64_t i = idx / ncols, col = col0 + idx % ncols;
    const uint64_t b = (band * pk::kBand + i) * g.bc + col;
    uint64_t start;
    int len;
    block_extent(s, b, start, len);
    BitWin bw;
    win_at(bw, s.words, start, len);
    Decoded d;
    decode_any<HAS_RAW>(s, bw, s.planes_limit, d);
    if (pk::is_exception(d)) {
      ++nexc;
      continue;
    }
    if (d.emax == 0) continue;
    emin = min(emin, d.emax);
    emx = max(emx, d.emax);
    int32_t q[16];
    pk::signed_coefs(d, q);
#pragma unroll
    for (int c = 0; c < 16; ++c) wmax[c] = max(wmax[c], (uint32_t)pk::qwidth(q[c]));
  }
  int W[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) W[c] = (int)__reduce_max_sync(0xFFFFFFFFu, wmax[c]);
  emin = __reduce_min_sync(0xFFFFFFFFu, emin);
  emx = __reduce_max_sync(0xFFFFFFFFu, emx);
  nexc = __reduce_add_sync(0xFFFFFFFFu, nexc);
  if (lane != 0) return;
  if (W[0] < 1) W[0] = 1;                  // the DC field is never empty
  const uint32_t ebase = emx >= emin ? emin : 0u;
  const int We = emx > emin ? pk::bitwidth_u(emx - emin) : 0;
  pk::Layout f;
  pk::make_layout(We, W, f);
  pk::Seg S;
  S.body = 0;
  S.hdr = pk::seg_hdr(ebase, f);
  S.w[0] = S.w[1] = S.w[2] = 0;
  S.o[0] = S.o[1] = S.o[2] = S.o[3] = 0;
  for (int c = 0; c < 16; ++c) {
    S.w[c / 6] |= (uint32_t)W[c] << (5 * (c % 6));
    if (f.fast) S.o[c / 4] |= (uint32_t)f.o[c] << (8 * (c % 4));
  }
  S.exc_begin = 0;
  S.exc_count = nexc;
  segs[sid] = S;
  seg_words[sid] = (uint64_t)pk::seg_tiles(g, sb) * pk::tile_words(f.L);
  seg_exc[sid] = nexc;
}

__global__ void k_pk_finalize(pk::Seg* segs, uint64_t nseg, const uint64_t* off, const uint64_t* eoff) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= nseg) return;
  segs[i].body = off[i];
  segs[i].exc_begin = (uint32_t)eoff[i];
}

// field widths / layout of a segment header
__device__ __forceinline__ void seg_layout(const pk::Seg& S, int W[16], pk::Layout& f) {
#pragma unroll
  for (int c = 0; c < 16; ++c) W[c] = pk::seg_W(S, c);
  pk::make_layout(pk::seg_We(S), W, f);
}

// ---------------------------------------------------------------------------
// packer, pass 2: records and exceptions
// ---------------------------------------------------------------------------
template <bool HAS_RAW>
__global__ void __launch_bounds__(256, WHFF_PK_MINB) k_pk_emit(StreamView s, pk::Geom g, const pk::Seg* segs,
                                                 uint32_t* body, uint64_t* exc_block,
                                                 uint32_t* exc_words) {
  const uint64_t sid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (sid >= g.nband * g.nsegb) return;
  const uint64_t band = sid / g.nsegb, sb = sid % g.nsegb;
  const int nrows = pk::band_rows(g, band);
  const pk::Seg S = segs[sid];
  int W[16];
  pk::Layout f;
  seg_layout(S, W, f);
  const int L = f.L, R = pk::rec_words(L);
  const uint32_t ebase = (uint32_t)pk::seg_emax_base(S);
  const uint64_t TW = pk::tile_words(L);
  uint64_t exc = S.exc_begin;
  const int ntl = pk::seg_tiles(g, sb);
  for (int tt = 0; tt < ntl; ++tt) {
    const uint64_t col = (sb * g.segt + tt) * pk::kTile + lane;
    const bool active = col < g.bc;
    for (int i = 0; i < nrows; ++i) {
      const uint64_t b = (band * pk::kBand + i) * g.bc + col;
      uint32_t rec[pk::kMaxRecordWords + 1];
#pragma unroll
      for (int k = 0; k <= pk::kMaxRecordWords; ++k) rec[k] = 0u;
      bool isexc = false;
      Decoded d;
      int32_t q[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) q[c] = 0;
      uint32_t ed = 0;
      if (active) {
        uint64_t start;
        int len;
        block_extent(s, b, start, len);
        BitWin bw;
        win_at(bw, s.words, start, len);
        decode_any<HAS_RAW>(s, bw, s.planes_limit, d);
        isexc = pk::is_exception(d);
        if (!isexc && d.emax != 0) {
          pk::signed_coefs(d, q);
          ed = d.emax - ebase;
        }
      }
      // zero blocks, exceptions and absent lanes: q = 0 (offset-binary 2^(W-1))
      pk::build_record(f, W, ed, q, rec);
      // word-major tile: word k of (row i, lane) at tile word (32 k + lane) * 4 + i
      uint32_t* tp = body + S.body + tt * TW;
      for (int k = 0; k < R; ++k) tp[pk::tile_word(k, lane, i)] = rec[k];
      // exceptions in (tile, row, lane) order
      const unsigned m = __ballot_sync(0xFFFFFFFFu, isexc);
      if (isexc) {
        const uint64_t e = exc + __popc(m & ((1u << lane) - 1u));
        exc_block[e] = b;
        float x[16];
        reconstruct_words(d, x);
#pragma unroll
        for (int k = 0; k < 16; ++k) exc_words[16 * e + k] = __float_as_uint(x[k]);
      }
      exc += __popc(m);
    }
  }
}

// per-segment parameter tables (after the headers): one thread per (segment, field)
__global__ void k_pk_params(const pk::Seg* segs, uint64_t nseg, pk::FieldPar* pars) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= nseg * 16) return;
  const pk::Seg S = segs[t >> 4];
  pars[t] = pk::seg_generic(S) ? pk::FieldPar{0u, 0u, 0u, 0u} : pk::seg_param(S, (int)(t & 15));
}

cudaError_t pk_launch_params(pk::Seg* segs, uint64_t nseg, cudaStream_t cs) {
  if (nseg) k_pk_params<<<grid_of(nseg * 16, 256), 256, 0, cs>>>(segs, nseg, reinterpret_cast<pk::FieldPar*>(segs + nseg));
  return cudaGetLastError();
}

cudaError_t pk_launch_stats(const StreamView& s, const pk::Geom& g, pk::Seg* segs, uint64_t* seg_words,
                            uint64_t* seg_exc, cudaStream_t cs) {
  const uint64_t nseg = g.nband * g.nsegb;
  if (s.has_raw) k_pk_stats<true><<<grid_of(nseg, 8), 256, 0, cs>>>(s, g, segs, seg_words, seg_exc);
  else k_pk_stats<false><<<grid_of(nseg, 8), 256, 0, cs>>>(s, g, segs, seg_words, seg_exc);
  return cudaGetLastError();
}

cudaError_t pk_launch_finalize(pk::Seg* segs, uint64_t nseg, const uint64_t* off, const uint64_t* eoff,
                               cudaStream_t cs) {
  k_pk_finalize<<<grid_of(nseg, 256), 256, 0, cs>>>(segs, nseg, off, eoff);
  return cudaGetLastError();
}

cudaError_t pk_launch_emit(const StreamView& s, const pk::Geom& g, const pk::Seg* segs, uint32_t* body,
                           uint64_t* exc_block, uint32_t* exc_words, cudaStream_t cs) {
  const uint64_t nseg = g.nband * g.nsegb;
  if (s.has_raw) k_pk_emit<true><<<grid_of(nseg, 8), 256, 0, cs>>>(s, g, segs, body, exc_block, exc_words);
  else k_pk_emit<false><<<grid_of(nseg, 8), 256, 0, cs>>>(s, g, segs, body, exc_block, exc_words);
  return cudaGetLastError();
}

