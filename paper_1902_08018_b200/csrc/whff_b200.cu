// whff_b200.cu -- sm_100a kernels and the C ABI of include/whff_b200.h.
//
// Hot path: k_decode_gemv, the fused WHFZ decode + mixed-precision GEMV
// (reference: codec.decompress (codec.py:296-314, K:371-408) followed by
// mpgemv.gemv(mixed, sequential) (mpgemv.py:54-61, K:24-47), as issued per
// light step by pipeline._compute_deltas (pipeline.py:199-205)).  One warp
// owns one 4-row block-row; lane l decodes block-columns l, l+32, ... so a
// warp's 32 segments are contiguous in HBM (coalesced 16-byte loads at
// FixedRate(8)); products accumulate per lane and reduce with a fixed xor
// butterfly: deterministic, no atomics.
//
// Everything else here (decode-only, decode_blocks parity hook, GPU encoder,
// dense GEMV policies, thermal CSR step) restates the reference operation
// named at each kernel.
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <type_traits>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/whff_b200.h"
#include "whff_decode.cuh"
#include "whff_encode.cuh"
#include "whff_relayout.cuh"
#include "whff_common.cuh"
#include "whff_packed_api.h"

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
namespace {
thread_local std::string g_err;

whff_status_t fail(whff_status_t s, const std::string& msg) {
  g_err = msg;
  return s;
}
whff_status_t cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? WHFF_ERR_NOMEM : WHFF_ERR_CUDA;
}
}  // namespace

#define WCK(x)                                             \
  do {                                                     \
    cudaError_t e_ = (x);                                  \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x);       \
  } while (0)
#define WCK_LAUNCH(what)                                   \
  do {                                                     \
    cudaError_t e_ = cudaGetLastError();                   \
    if (e_ != cudaSuccess) return cuda_fail(e_, what);     \
  } while (0)

struct whff_dstream {
  int device;
  int mode;
  double param;
  uint64_t rows, cols, br, bc, nb, gpr;
  uint64_t payload_bytes, payload_bits, total_bits = 0;
  int planes_limit, has_raw, kind;
  int layout = WHFF_LAYOUT_REFERENCE;
  uint32_t seg_bits;
  uint8_t* d_payload = nullptr;
  size_t payload_alloc = 0;
  uint64_t* d_base = nullptr;
  uint16_t* d_lens = nullptr;
  uint64_t* d_starts = nullptr;
  size_t index_bytes = 0;
  // tile-packed representation (whff_dstream_pack; whff_packed.cuh)
  bool packed = false;
  uint32_t* d_pk_body = nullptr;
  pk::Seg* d_pk_segs = nullptr;
  uint64_t* d_pk_exc_block = nullptr;
  uint32_t* d_pk_exc_words = nullptr;
  uint64_t pk_body_words = 0, pk_nexc = 0, pk_alloc_words = 0;
  std::vector<uint64_t> pk_band_bytes;   // bytes a GEMV reads per band (body + headers + exceptions)

  StreamView view() const {
    StreamView v;
    v.words = reinterpret_cast<const uint32_t*>(d_payload);
    v.base = d_base;
    v.lens = d_lens;
    v.starts = d_starts;
    v.payload_bits = payload_bits;
    v.rows = rows;
    v.cols = cols;
    v.br = br;
    v.bc = bc;
    v.gpr = gpr;
    v.seg_bits = seg_bits;
    v.kind = kind;
    v.planes_limit = planes_limit;
    v.has_raw = has_raw;
    v.layout = layout;
    return v;
  }
};

// ---------------------------------------------------------------------------
// decode_blocks parity hook (K:371-408)
// ---------------------------------------------------------------------------
template <bool HAS_RAW>
__global__ void __launch_bounds__(128) k_decode_blocks(StreamView s, uint64_t first, uint64_t count,
                                                       int planes_limit, uint32_t* mag, uint8_t* neg,
                                                       uint16_t* emax, uint8_t* raw,
                                                       uint32_t* raw_words, uint64_t* consumed) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint64_t b = first + i;
  uint64_t start;
  int len;
  block_extent(s, b, start, len);
  BitWin bw;
  win_at(bw, s.words, start, len);
  Decoded d;
  decode_any<HAS_RAW>(s, bw, planes_limit, d);
  emax[i] = (uint16_t)d.emax;
  raw[i] = (uint8_t)d.raw;
  consumed[i] = (uint64_t)d.consumed;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    mag[16 * i + c] = d.raw ? 0u : d.mag[c];
    raw_words[16 * i + c] = d.raw ? d.mag[c] : 0u;
    neg[16 * i + c] = (uint8_t)((d.negm >> c) & 1u);
  }
}

// ---------------------------------------------------------------------------
// reconstructed blocks (codec.py:209-218), the device half of decode_block
// ---------------------------------------------------------------------------
template <bool HAS_RAW>
__global__ void __launch_bounds__(128) k_decode_block_words(StreamView s, uint64_t first, uint64_t count,
                                                            float* out) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  uint64_t start;
  int len;
  block_extent(s, first + i, start, len);
  BitWin bw;
  win_at(bw, s.words, start, len);
  Decoded d;
  decode_any<HAS_RAW>(s, bw, s.planes_limit, d);
  float x[16];
  reconstruct_words(d, x);
#pragma unroll
  for (int c = 0; c < 16; ++c) out[16 * i + c] = x[c];
}

// ---------------------------------------------------------------------------
// decompress (codec.py:296-314): bit-exact words, non-finite -> status
// ---------------------------------------------------------------------------
// One warp per group of 32 consecutive blocks of a block-row (the fused
// kernel's organisation): the compact index is resolved with one shuffle scan
// per warp, the in-register window is used whenever every lane's segment fits
// it, and the layout is a template parameter.
template <bool HAS_RAW, bool SF>
__global__ void __launch_bounds__(256) k_decode_words(StreamView s, float* out, uint64_t ld,
                                                      unsigned long long* status) {
  const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= s.br * s.gpr) return;                   // warp-uniform
  const uint64_t brow = wid / s.gpr, g = wid - brow * s.gpr;
  const uint64_t bcol = g * 32 + lane;
  const bool active = bcol < s.bc;
  const uint64_t b = brow * s.bc + bcol;
  uint64_t start = 0;
  int len = 0;
  if (s.kind == WHFF_INDEX_COMPACT) {
    const uint32_t l = active ? (uint32_t)s.lens[b] : 0u;
    uint32_t incl = l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += t;
    }
    start = s.base[brow * s.gpr + g] + (incl - l);
    if (active) len = clamp_len(start, l, s.payload_bits);
  } else if (active) {
    block_extent(s, b, start, len);
  }
  BitWin bw;
  if (active) {
    win_at(bw, s.words, start, len);
  } else {
    bw.w0 = bw.w1 = bw.w2 = bw.w3 = 0u;
    bw.pos = 0;
    bw.len = 0;
    bw.avail = 128;
    bw.src = s.words;
  }
  Decoded d;
  if (__any_sync(0xFFFFFFFFu, active && !fits_no_refill(start, len))) {
    if (SF) decode_block_sf<HAS_RAW, true>(bw, s.planes_limit, d);
    else decode_block<HAS_RAW, true>(bw, s.planes_limit, d, 0xFFFFFFFFu);
  } else {
    if (SF) decode_block_sf<HAS_RAW, false>(bw, s.planes_limit, d);
    else decode_block<HAS_RAW, false>(bw, s.planes_limit, d, 0xFFFFFFFFu);
  }
  if (!active) return;
  float x[16];
  reconstruct_words(d, x);
  const uint64_t r0 = brow * 4, c0 = bcol * 4;
  // interior blocks of a 16-byte aligned output: one 16-byte store per row
  const bool full = r0 + 4 <= s.rows && c0 + 4 <= s.cols &&
                    ((reinterpret_cast<uintptr_t>(out) | (ld * 4)) & 15u) == 0;
  if (full) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      *reinterpret_cast<float4*>(out + (r0 + i) * ld + c0) =
          make_float4(x[4 * i], x[4 * i + 1], x[4 * i + 2], x[4 * i + 3]);
    uint32_t anybad = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) anybad |= (__float_as_uint(x[k]) & 0x7F800000u) == 0x7F800000u;
    if (!anybad) return;
  }
  unsigned long long bad = ~0ull;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint64_t r = r0 + i;
    if (r >= s.rows) break;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t c = c0 + j;
      if (c < s.cols) {
        if (!full) out[r * ld + c] = x[4 * i + j];
        if (!isfinite(x[4 * i + j])) {
          const unsigned long long f = r * s.cols + c;
          bad = f < bad ? f : bad;
        }
      }
    }
  }
  if (bad != ~0ull) atomicMin(status, bad);
}

// ---------------------------------------------------------------------------
// Fused decode + GEMV (the hot path)
// ---------------------------------------------------------------------------
struct GemvJob {
  StreamView s;
  const float* v;
  const float4* U;     // coefficient domain: G^T v per block-column
  float* y;
  uint64_t row_begin, row_end;
  uint64_t br0;        // first block-row of the job
};

// Per-virtual-warp partial sums of one block-row (see k_decode_gemv).
struct VwRec {
  double d[4];
  double r[4];
  float f[4];
  float rf[4];
  float probe;
  float pad;
};

struct JobTable {
  const GemvJob* jobs;       // device table (plans) or nullptr
  const uint64_t* prefix;    // first block-row of each job
  const uint32_t* row_job;   // job of each block-row
  int n;
  uint64_t total_warps;      // block-rows
  GemvJob single;            // used when jobs == nullptr
  VwRec* recs;               // [block-row][kVW] partials
  unsigned* tickets;         // [block-row] warp arrival counters (zero between launches)
};

// Accumulators for the three policies (mpgemv.py:1-7):
//   mixed : binary32 product, binary64 sum     single: binary32 both
//   double: binary64 product and sum
struct Acc {
  double d[4];
  float f[4];
  float probe;   // single policy: NaN iff a decoded value was non-finite
};

__device__ __forceinline__ void acc_exact(Acc& A, int policy, const float x_in[16], float4 v4,
                                          uint32_t colmask) {
  const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
  float x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = x_in[k];
  if (colmask != 0xFu) {          // last block-column: padded columns contribute nothing
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (!((colmask >> (k & 3)) & 1u)) x[k] = 0.0f;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float xv = x[4 * i + j];
      if (policy == WHFF_POLICY_MIXED) {
        A.d[i] = __dadd_rn(A.d[i], (double)__fmul_rn(xv, vv[j]));
      } else if (policy == WHFF_POLICY_SINGLE) {
        A.f[i] = __fadd_rn(A.f[i], __fmul_rn(xv, vv[j]));
        A.probe = __fmaf_rn(xv, 0.0f, A.probe);
      } else {
        A.d[i] = __dadd_rn(A.d[i], __dmul_rn((double)xv, (double)vv[j]));
      }
    }
  }
}

// coefficient domain: w = Q u (Q at raster positions), acc += 2^k w
__device__ __forceinline__ void acc_coeff(Acc& A, int policy, const Decoded& d, float4 u4, int k) {
  const float u[4] = {u4.x, u4.y, u4.z, u4.w};
  float w[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const int pos = seq_pos(c);
    float q = (float)d.mag[c];
    q = ((d.negm >> c) & 1u) ? -q : q;
    w[pos >> 2] = __fmaf_rn(q, u[pos & 3], w[pos >> 2]);
  }
  const float s = scale_f32(k);
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const float t = __fmul_rn(w[a], s);
    if (policy == WHFF_POLICY_SINGLE) A.f[a] = __fadd_rn(A.f[a], t);
    else A.d[a] = __dadd_rn(A.d[a], (double)t);
  }
}

// Coefficient-domain accumulator fed by the fields loop of decode_block_sf:
// w[r] += q_c * u[j] for each significant coefficient c at raster (r, j),
// in coefficient order (identical arithmetic to acc_coeff, which also adds
// the zero coefficients as exact no-ops).
// blocks the coefficient domain evaluates (zero blocks trivially): not a raw
// escape, and a scale 2^k with k in [-126, 100] (no fp32 over/underflow)
__device__ __forceinline__ bool coef_ok(const Decoded& d) {
  const int k = (int)d.emax - kEmaxBias - kQuantBits;
  return !d.raw && (d.emax == 0 || (k >= -126 && k <= 100));
}

struct CoefSink {
  float u[4];
  float w[4];
  template <int C>
  __device__ __forceinline__ void coef(uint32_t mag, uint32_t sign31) {   // sign at bit 31
    constexpr int pos = seq_pos(C);
    float q = __uint2float_rn(mag);
    q = __uint_as_float(__float_as_uint(q) ^ (sign31 & 0x80000000u));
    w[pos >> 2] = __fmaf_rn(q, u[pos & 3], w[pos >> 2]);
  }
};

// Coefficient-domain kernels: the rare blocks coef_ok() rejects (raw
// escapes, extreme scales) are re-decoded here with their exact words and
// accumulated in the spatial domain.  Out of line so the hot loop keeps its
// register budget (64) and its instruction footprint.
template <bool HAS_RAW>
__device__ __noinline__ void coef_fallback(const uint32_t* words, uint64_t start, int len, int pl,
                                           const float* v, uint64_t bcol, uint64_t cols,
                                           bool v_aligned, uint32_t colmask, int policy, Acc* R) {
  BitWin bw;
  win_at(bw, words, start, len);
  Decoded d;
  decode_block_sf<HAS_RAW, true>(bw, pl, d);
  if (!d.raw && d.emax == 0) return;
  const float4 v4 = load_v4(v, bcol, cols, v_aligned);
  float x[16];
  reconstruct_words(d, x);
  acc_exact(*R, policy, x, v4, colmask);
}

constexpr int kGemvWarps = 8;
// A block-row's 32-block groups are summed in kVW "virtual warps": virtual
// warp w takes groups w, w + kVW, w + 2 kVW, ... (one partial per lane, then
// a fixed butterfly).  Each row runs on kSplit CTAs of 8 warps (one virtual
// warp per warp), so launches with few block-rows (a light step: 3 slits =
// 285 rows) still fill the GPU; the last of the row's warps to finish adds
// the kVW partials with another fixed butterfly.  The order is fixed, so a
// row's result does not depend on the launch that computes it.
constexpr int kSplit = kVW / kGemvWarps;   // CTAs per block-row

// Software-pipelined segment location for indexed / implicit variable-rate
// streams (see k_decode_gemv).  Holds, for the next group, its start bit,
// length and first four payload words, and for the group after it the
// lane's raw index entries.
template <bool INDEXED>
struct SegPrefetch {
  uint64_t start = 0;
  int len = 0;
  uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  uint32_t il = 0;      // index entries of group gi (lens / starts, base)
  uint64_t ib = 0;

  __device__ __forceinline__ void load_index(const StreamView& s, uint64_t brow, uint64_t row_block0,
                                             uint64_t bc, uint64_t gi, int lane) {
    if (!INDEXED || gi >= s.gpr) return;
    const uint64_t bcol = gi * 32 + lane;
    const bool act = bcol < bc;
    const uint64_t b = row_block0 + bcol;
    il = act ? (uint32_t)s.lens[b] : 0u;
    if (s.kind == WHFF_INDEX_COMPACT) ib = s.base[brow * s.gpr + gi];
    else ib = act ? s.starts[b] : 0ull;
  }
  // locate group gn (its index entries are in il/ib) and load its words
  __device__ __forceinline__ void locate(const StreamView& s, uint64_t row_block0, uint64_t bc,
                                         uint64_t gn, int lane) {
    if (gn >= s.gpr) return;                 // warp-uniform
    const uint64_t bcol = gn * 32 + lane;
    const bool act = bcol < bc;
    const uint64_t b = row_block0 + bcol;
    len = 0;
    if (!INDEXED) {
      start = b * (uint64_t)s.seg_bits;
      if (act) len = clamp_len(start, s.seg_bits, s.payload_bits);
    } else if (s.kind == WHFF_INDEX_COMPACT) {
      uint32_t incl = il;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += t;
      }
      start = ib + (incl - il);
      if (act) len = clamp_len(start, il, s.payload_bits);
    } else {
      start = ib;
      if (act) len = clamp_len(start, il, s.payload_bits);
    }
    if (act) {
      const uint32_t* p = s.words + (start >> 5);
      a0 = ldg(p); a1 = ldg(p + 1); a2 = ldg(p + 2); a3 = ldg(p + 3);
    }
  }
  // a warp's groups are g0, g0 + kVW, g0 + 2 kVW, ... (see kVW)
  __device__ __forceinline__ void prologue(const StreamView& s, uint64_t brow, uint64_t row_block0,
                                           uint64_t bc, uint64_t g0, int lane) {
    load_index(s, brow, row_block0, bc, g0, lane);
    locate(s, row_block0, bc, g0, lane);
    load_index(s, brow, row_block0, bc, g0 + kVW, lane);
  }
  // called at group g with gn = g + kVW: locate gn, fetch the index of gn + kVW
  __device__ __forceinline__ void advance(const StreamView& s, uint64_t brow, uint64_t row_block0,
                                          uint64_t bc, uint64_t gn, int lane) {
    locate(s, row_block0, bc, gn, lane);
    load_index(s, brow, row_block0, bc, gn + kVW, lane);
  }
};

template <int VAR>
struct VarTraits;
// 0: FixedRate(8) implicit index, one 16-byte load per block, no refill
template <> struct VarTraits<0> { static constexpr bool kRefill = false, kRaw = false, kIndexed = false; };
// 1: any implicit fixed rate
template <> struct VarTraits<1> { static constexpr bool kRefill = true, kRaw = false, kIndexed = false; };
// 2: indexed (compact/full), no raw flag (fixed precision / odd rate offsets)
template <> struct VarTraits<2> { static constexpr bool kRefill = true, kRaw = false, kIndexed = true; };
// 3: indexed with raw flag (fixed accuracy)
template <> struct VarTraits<3> { static constexpr bool kRefill = true, kRaw = true, kIndexed = true; };

// launch bounds: fixed-rate variants are held at 64 registers (4 CTAs/SM),
// measured best for the fused kernel; the indexed ones settle at 74-80 (3
// CTAs/SM) on their own; -DWHFF_GEMV_MINB=n overrides for sweeps
#ifdef WHFF_GEMV_MINB
#define WHFF_GEMV_LB __launch_bounds__(256, WHFF_GEMV_MINB)
#else
#define WHFF_GEMV_LB __launch_bounds__(256, VAR <= 1 ? 4 : 3)
#endif

template <int VAR, int EVAL, bool SF, int POL>
__global__ void WHFF_GEMV_LB k_decode_gemv(JobTable T, unsigned long long* status) {
  using TR = VarTraits<VAR>;
  constexpr int policy = POL;   // compile-time: only the policy's accumulators exist
  // kSplit CTAs per (job, block-row); warp w of CTA part q runs the row's
  // virtual warp 8 q + w (see kVW)
  const uint64_t gr = blockIdx.x / kSplit;
  const int part = (int)(blockIdx.x % kSplit);
  if (gr >= T.total_warps) return;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  uint64_t first_row = 0;
  int jidx = -1;
  if (T.jobs != nullptr) {
    if (VAR == 0) {           // (the search measured faster here than the table, by codegen)
      int lo = 0, hi = T.n - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (T.prefix[mid] <= gr) lo = mid; else hi = mid - 1;
      }
      jidx = lo;
    } else {
      jidx = (int)T.row_job[gr];
    }
    first_row = T.prefix[jidx];
  }
  const StreamView s = jidx < 0 ? T.single.s : T.jobs[jidx].s;
  const float* __restrict__ v = jidx < 0 ? T.single.v : T.jobs[jidx].v;
  const float4* __restrict__ U = jidx < 0 ? T.single.U : T.jobs[jidx].U;
  float* __restrict__ yout = jidx < 0 ? T.single.y : T.jobs[jidx].y;
  const uint64_t row_begin = jidx < 0 ? T.single.row_begin : T.jobs[jidx].row_begin;
  const uint64_t row_end = jidx < 0 ? T.single.row_end : T.jobs[jidx].row_end;
  const uint64_t br0 = jidx < 0 ? T.single.br0 : T.jobs[jidx].br0;
  const uint64_t brow = br0 + (gr - first_row);
  const uint64_t bc = s.bc;
  const bool v_aligned = ((reinterpret_cast<uintptr_t>(v) & 15u) == 0);
  const uint32_t last_colmask = (s.cols & 3) ? ((1u << (s.cols & 3)) - 1u) : 0xFu;
  const int pl = s.planes_limit;

  Acc A;
#pragma unroll
  for (int i = 0; i < 4; ++i) { A.d[i] = 0.0; A.f[i] = 0.0f; }
  A.probe = 0.0f;
  // coefficient domain: spatial part of the rare raw / extreme-scale blocks.
  // Its address goes to the out-of-line fallback, so it lives in memory: in
  // shared memory, since a local-memory frame zeroed by every thread of every
  // CTA was written back to HBM (0.95 GB per config-3 step).
  __shared__ Acc s_rs[32 * kGemvWarps];
  Acc& RS = s_rs[threadIdx.x];
#pragma unroll
  for (int i = 0; i < 4; ++i) { RS.d[i] = 0.0; RS.f[i] = 0.0f; }
  RS.probe = 0.0f;

  // this warp's groups: vw, vw + kVW, ... (< gpr)
  const int vw = part * kGemvWarps + warp;

  const uint64_t row_block0 = brow * bc;
  const uint4* __restrict__ seg128 = reinterpret_cast<const uint4*>(s.words);
  uint4 nxt = make_uint4(0, 0, 0, 0);
  // FixedRate(8): the payload covers this block-row's segments completely
  const bool row_full = VAR == 0 && (row_block0 + bc) * 128ull <= s.payload_bits;
  if (VAR == 0) {
    const uint64_t bcol0 = (uint64_t)vw * 32 + lane;
    if (bcol0 < bc) nxt = ldg(seg128 + row_block0 + bcol0);
  }
  // Variable-length streams: the segment of the next group is located (index
  // loaded one iteration earlier) and its four payload words are loaded
  // while group g decodes; the index of the group after is loaded meanwhile.
  SegPrefetch<TR::kIndexed> pf;
  if (VAR != 0) pf.prologue(s, brow, row_block0, bc, (uint64_t)vw, lane);

  // (32-bit group index for FixedRate(8): measured fewer instructions)
  using GI = typename std::conditional<VAR == 0, uint32_t, uint64_t>::type;
  for (GI g = vw; g < (GI)s.gpr; g += kVW) {
    const uint64_t bcol = (uint64_t)g * 32 + lane;
    const bool active = bcol < bc;
    const uint64_t b = row_block0 + bcol;
    BitWin bw;
    Decoded d;
    uint64_t fb_start = b * 128ull;          // the block's segment (coefficient fallback)
    int fb_len = 0;
    // coefficient domain + skeleton-first: accumulate inside the fields loop
    constexpr bool kSink = SF && EVAL == WHFF_EVAL_COEFF;
    CoefSink cs;
    if (kSink) {
      const float4 u4 = active ? ldg(U + bcol) : make_float4(0.f, 0.f, 0.f, 0.f);
      cs.u[0] = u4.x; cs.u[1] = u4.y; cs.u[2] = u4.z; cs.u[3] = u4.w;
#pragma unroll
      for (int a = 0; a < 4; ++a) cs.w[a] = 0.0f;
    }
    if (VAR == 0) {
      const uint4 q = nxt;
      const uint64_t bn = bcol + 32 * kVW;
      if (bn < bc) nxt = ldg(seg128 + row_block0 + bn);   // prefetch this warp's next group
      if (row_full) {                        // every segment of the row is whole: no masks
        fb_len = 128;                        // (lanes past the row end decode zeros, discarded)
        win_128(bw, q.x, q.y, q.z, q.w, 128);
      } else {
        fb_len = active ? clamp_len(b * 128ull, 128ull, s.payload_bits) : 0;
        win_128(bw, q.x, q.y, q.z, q.w, fb_len);
      }
      if (kSink) decode_block_sf<false, false, CoefSink&, false, false>(bw, pl, d, cs);
      else if (SF) decode_block_sf<false, false, NullSink, true, false>(bw, pl, d);
      else decode_block<false, false, false>(bw, pl, d, 0xFFFFFFFFu);
    } else {
      const uint64_t start = pf.start;
      const int len = pf.len;
      const uint32_t a0 = pf.a0, a1 = pf.a1, a2 = pf.a2, a3 = pf.a3;
      pf.advance(s, brow, row_block0, bc, g + kVW, lane);
      if (active) {
        win_words(bw, s.words, start, len, a0, a1, a2, a3);
      } else {
        bw.w0 = bw.w1 = bw.w2 = bw.w3 = 0u;
        bw.pos = 0;
        bw.len = 0;
        bw.avail = 128;
        bw.src = s.words;
      }
      fb_start = start;
      fb_len = len;
      if (__any_sync(0xFFFFFFFFu, active && !fits_no_refill(start, len))) {
        if (kSink) decode_block_sf<TR::kRaw, true, CoefSink&, false>(bw, pl, d, cs);
        else if (SF) decode_block_sf<TR::kRaw, true>(bw, pl, d);
        else decode_block<TR::kRaw, true>(bw, pl, d, 0xFFFFFFFFu);
      } else {
        if (kSink) decode_block_sf<TR::kRaw, false, CoefSink&, false>(bw, pl, d, cs);
        else if (SF) decode_block_sf<TR::kRaw, false>(bw, pl, d);
        else decode_block<TR::kRaw, false>(bw, pl, d, 0xFFFFFFFFu);
      }
    }
    if (!active) continue;
    const uint32_t colmask = (bcol + 1 == bc) ? last_colmask : 0xFu;

    if (EVAL == WHFF_EVAL_EXACT) {
      const float4 v4 = load_v4(v, bcol, s.cols, v_aligned);
      float x[16];
      reconstruct_words(d, x);
      acc_exact(A, policy, x, v4, colmask);
    } else {
      const int k = (int)d.emax - kEmaxBias - kQuantBits;
      if (kSink && !coef_ok(d)) {
        coef_fallback<TR::kRaw>(s.words, fb_start, fb_len, pl, v, bcol, s.cols, v_aligned, colmask,
                                policy, &RS);
      } else if (coef_ok(d) && d.emax != 0) {
        if (kSink) {
          const float sc = scale_f32(k);
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const float t = __fmul_rn(cs.w[a], sc);
            if (policy == WHFF_POLICY_SINGLE) A.f[a] = __fadd_rn(A.f[a], t);
            else A.d[a] = __dadd_rn(A.d[a], (double)t);
          }
        } else {
          acc_coeff(A, policy, d, ldg(U + bcol), k);
        }
      } else if (d.raw || d.emax != 0) {   // raw escape / extreme scale: exact spatial path
        const float4 v4 = load_v4(v, bcol, s.cols, v_aligned);
        float x[16];
        reconstruct_words(d, x);
        acc_exact(RS, policy, x, v4, colmask);
      }
    }
  }

  double accR[4];
  float accRf[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) { accR[i] = RS.d[i]; accRf[i] = RS.f[i]; }
  if (EVAL == WHFF_EVAL_COEFF) A.probe = __fadd_rn(A.probe, RS.probe);
  // fixed xor butterfly over the warp (only the policy's accumulators)
  constexpr bool kF = policy == WHFF_POLICY_SINGLE, kD = !kF, kC = EVAL == WHFF_EVAL_COEFF;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (kD) A.d[i] = __dadd_rn(A.d[i], __shfl_xor_sync(0xFFFFFFFFu, A.d[i], o));
      if (kF) A.f[i] = __fadd_rn(A.f[i], __shfl_xor_sync(0xFFFFFFFFu, A.f[i], o));
      if (kC && kD) accR[i] = __dadd_rn(accR[i], __shfl_xor_sync(0xFFFFFFFFu, accR[i], o));
      if (kC && kF) accRf[i] = __fadd_rn(accRf[i], __shfl_xor_sync(0xFFFFFFFFu, accRf[i], o));
    }
    if (kF) A.probe = __fadd_rn(A.probe, __shfl_xor_sync(0xFFFFFFFFu, A.probe, o));
  }
  // publish this virtual warp's partials; the last of the row's kVW warps to
  // finish adds the kVW partials (fixed xor butterfly) and writes the rows
  // (row and virtual warp recomputed: nothing extra stays live across the loop)
  VwRec* grec = T.recs + (uint64_t)(blockIdx.x / kSplit) * kVW;
  unsigned last = 0;
  if (lane == 0) {
    VwRec R;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      R.d[i] = A.d[i];
      R.f[i] = A.f[i];
      R.r[i] = EVAL == WHFF_EVAL_COEFF ? accR[i] : 0.0;
      R.rf[i] = EVAL == WHFF_EVAL_COEFF ? accRf[i] : 0.0f;
    }
    R.probe = A.probe;
    R.pad = 0.0f;
    grec[(blockIdx.x % kSplit) * kGemvWarps + (threadIdx.x >> 5)] = R;
    // release: the record is visible before the count (no full fence: a
    // gpu-scope __threadfence per warp also invalidated the SM's L1)
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.inc.u32 %0, [%1], %2;"
                 : "=r"(old) : "l"(T.tickets + blockIdx.x / kSplit), "r"(kVW - 1u) : "memory");
    last = old == kVW - 1u;
  }
  if (!__shfl_sync(0xFFFFFFFFu, last, 0)) return;
  // lane 0's acquire covers the warp once the warp synchronises (the shuffle
  // alone carries no memory ordering to lanes 1..31)
  __syncwarp();
  asm volatile("fence.acq_rel.gpu;" ::: "memory");   // the other warps' records (read via L2)
  VwRec P;
  {
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(grec + lane);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(&P);
#pragma unroll
    for (int k = 0; k < (int)(sizeof(VwRec) / 8); ++k) dst[k] = __ldcg(src + k);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      if (kD) P.d[a] = __dadd_rn(P.d[a], __shfl_xor_sync(0xFFFFFFFFu, P.d[a], o));
      if (kF) P.f[a] = __fadd_rn(P.f[a], __shfl_xor_sync(0xFFFFFFFFu, P.f[a], o));
      if (kC && kD) P.r[a] = __dadd_rn(P.r[a], __shfl_xor_sync(0xFFFFFFFFu, P.r[a], o));
      if (kC && kF) P.rf[a] = __fadd_rn(P.rf[a], __shfl_xor_sync(0xFFFFFFFFu, P.rf[a], o));
    }
    if (kF) P.probe = __fadd_rn(P.probe, __shfl_xor_sync(0xFFFFFFFFu, P.probe, o));
  }
  if (lane < 4) {
    const int i = lane;
    double td[4], tR = 0.0;
    float tf[4], tRf = 0.0f;
    const float probe = P.probe;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      td[a] = P.d[a];
      tf[a] = P.f[a];
      if (a == i) { tR = P.r[a]; tRf = P.rf[a]; }
    }
    const uint64_t r = brow * 4 + i;
    if (r >= row_begin && r < row_end && r < s.rows) {
      float out;
      bool bad;
      if (EVAL == WHFF_EVAL_EXACT) {
        if (policy == WHFF_POLICY_SINGLE) {
          out = tf[i];
          bad = !isfinite(probe);
        } else {
          out = __double2float_rn(td[i]);
          bad = !isfinite(td[i]);
        }
      } else {
        if (policy == WHFF_POLICY_SINGLE) {
          float t = tRf;
#pragma unroll
          for (int a = 0; a < 4; ++a) t = __fmaf_rn(c_G[i][a], tf[a], t);
          out = t;
          bad = !isfinite(probe);
        } else {
          double t = tR;
#pragma unroll
          for (int a = 0; a < 4; ++a) t = __fma_rn((double)c_G[i][a], td[a], t);
          out = __double2float_rn(t);
          bad = !isfinite(t);
        }
      }
      yout[r - row_begin] = out;
      if (bad) atomicMin(status, (unsigned long long)r);
    }
  }
}

// u_b = G^T v_b per block-column (coefficient-domain prologue)
// U = G^T v per block-column, zero-padded to whole 32-column tiles (bcp)
static uint64_t pad_tiles(uint64_t bc) { return (bc + 31) & ~31ull; }
__global__ void k_coeff_prep(const float* v, uint64_t cols, uint64_t bc, uint64_t bcp, float4* U) {
  const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (b >= bcp) return;
  if (b >= bc) {
    U[b] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const float4 x = load_v4(v, b, cols, false);
  const float xv[4] = {x.x, x.y, x.z, x.w};
  float u[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) t += (double)c_G[j][k] * (double)xv[j];
    u[k] = (float)t;
  }
  U[b] = make_float4(u[0], u[1], u[2], u[3]);
}

// v per block-column as float4, zero-padded past cols and to whole 32-column
// tiles (the staged exact evaluation copies it in tile slices like U)
__global__ void k_vpad(const float* v, uint64_t cols, uint64_t bc, uint64_t bcp, float4* V) {
  const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (b >= bcp) return;
  V[b] = b < bc ? load_v4(v, b, cols, false) : make_float4(0.f, 0.f, 0.f, 0.f);
}

// ---------------------------------------------------------------------------
// Dense GEMV policies (K:24-132)
// ---------------------------------------------------------------------------
// strict left-to-right per row (K:24-47); one thread per row.
template <int POL, bool F64OUT>
__global__ void k_gemv_seq(const float* A, uint64_t lda, uint64_t rows, uint64_t cols,
                           const float* v, float* y, double* y64) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const float* row = A + i * lda;
  if (POL == WHFF_POLICY_SINGLE) {
    float acc = 0.0f;
    for (uint64_t j = 0; j < cols; ++j) acc = __fadd_rn(acc, __fmul_rn(row[j], ldg(v + j)));
    y[i] = acc;
  } else {
    double acc = 0.0;
    for (uint64_t j = 0; j < cols; ++j) {
      const double p = POL == WHFF_POLICY_DOUBLE ? __dmul_rn((double)row[j], (double)ldg(v + j))
                                                 : (double)__fmul_rn(row[j], ldg(v + j));
      acc = __dadd_rn(acc, p);
    }
    if (F64OUT) y64[i] = acc;
    else y[i] = __double2float_rn(acc);
  }
}

// The same strict left-to-right order, one lane per row, fed by bulk copies.
// Each row is a serial chain of adds: on B200 a dependent binary64 add is 8
// cycles, and a conversion or product feeding it makes 13 (mixed) to 18
// (double) cycles per element from registers (5 for single), so the
// kernel's floor is cols x that, and everything else must stay off the
// chain.  Each warp owns `nr` <= 32 rows and its own ring of kSqStages
// shared-memory stages; a stage holds a sq_cols(nr)-column slice of each of
// the warp's rows (one cp.async.bulk per lane, rows padded to an odd number
// of 16-byte chunks so the lanes' 16-byte reads do not conflict) and the
// matching slice of v, all completing on the stage's mbarrier.  Four warps
// per CTA, one per SM sub-partition, and `nr` chosen so the warps cover the
// 148 x 4 sub-partitions once: two chains on one sub-partition would share
// its FP64 pipe and run at half speed.  Needs A, v 16-byte aligned and
// lda % 4 == 0; the last cols % 4 columns are read from global memory.
constexpr int kSqStages = 4;
constexpr int kSqWarps = 4;
// columns per stage (a multiple of 8: odd 16-byte row stride)
__host__ __device__ constexpr int sq_cols(int nr) {
  return nr <= 1 ? 1024 : nr <= 2 ? 512 : nr <= 4 ? 256 : nr <= 8 ? 128 : 64;
}
__host__ __device__ constexpr int sq_row_bytes(int nr) { return sq_cols(nr) * 4 + 16; }
__host__ __device__ constexpr int sq_stage_bytes(int nr) { return nr * sq_row_bytes(nr) + sq_cols(nr) * 4; }
__host__ __device__ constexpr int sq_warp_bytes(int nr) {
  return (kSqStages * sq_stage_bytes(nr) + kSqStages * 8 + 127) / 128 * 128;
}

template <int POL>
__global__ void __launch_bounds__(32 * kSqWarps) k_gemv_seq_staged(const float* A, uint64_t lda, uint64_t rows,
                                                                   uint64_t cols, const float* v, float* y, int nr) {
  extern __shared__ __align__(128) uint8_t sq_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t r0 = ((uint64_t)blockIdx.x * kSqWarps + warp) * nr;
  if (r0 >= rows) return;
  const int nrow = rows - r0 < (uint64_t)nr ? (int)(rows - r0) : nr;
  const int rl = lane < nrow ? lane : 0;   // idle lanes shadow the first row
  const int sb = sq_stage_bytes(nr), kc = sq_cols(nr), rb = sq_row_bytes(nr);
  const uint32_t st0 = (uint32_t)__cvta_generic_to_shared(sq_smem) + warp * sq_warp_bytes(nr);
  const uint32_t bar0 = st0 + kSqStages * sb;
  const uint32_t voff = nr * rb;
  const uint64_t cmain = cols & ~3ull;
  const uint64_t nchunk = (cmain + kc - 1) / kc;
  if (lane == 0)
    for (int s = 0; s < kSqStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * s) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto issue = [&](uint64_t c) {
    if (c >= nchunk) return;
    const int s = (int)(c % kSqStages);
    const uint64_t j0 = c * kc;
    const uint32_t bytes = (uint32_t)((cmain - j0 < (uint64_t)kc ? cmain - j0 : (uint64_t)kc) * 4);
    const uint32_t st = st0 + s * sb, bar = bar0 + 8 * s;
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes * (nrow + 1))
                   : "memory");
    __syncwarp();
    if (lane < nrow)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(st + lane * rb), "l"(A + (r0 + lane) * lda + j0), "r"(bytes), "r"(bar)
                   : "memory");
    if (lane == 0)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(st + voff), "l"(v + j0), "r"(bytes), "r"(bar)
                   : "memory");
  };
  for (int s = 0; s < kSqStages; ++s) issue(s);
  using AT = typename std::conditional<POL == WHFF_POLICY_SINGLE, float, double>::type;
  AT acc = 0;
  auto add = [&](float a, float b) {
    if (POL == WHFF_POLICY_SINGLE) acc = __fadd_rn(acc, __fmul_rn(a, b));
    else if (POL == WHFF_POLICY_MIXED) acc = __dadd_rn(acc, (double)__fmul_rn(a, b));
    else acc = __dadd_rn(acc, __dmul_rn((double)a, (double)b));
  };
  auto lds4 = [&](uint32_t addr) {
    float4 r;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "r"(addr));
    return r;
  };
  auto add4 = [&](const float4& a, const float4& b) {
    add(a.x, b.x);
    add(a.y, b.y);
    add(a.z, b.z);
    add(a.w, b.w);
  };
  for (uint64_t c = 0; c < nchunk; ++c) {
    const int s = (int)(c % kSqStages);
    const uint32_t phase = (uint32_t)((c / kSqStages) & 1);
    const uint32_t bar = bar0 + 8 * s;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "SQ_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra SQ_WAIT_%=;\n"
        "}\n" ::"r"(bar), "r"(phase) : "memory");
    const uint32_t ra = st0 + s * sb + rl * rb, va = st0 + s * sb + voff;
    const int n4 = (int)((cmain - c * kc < (uint64_t)kc ? cmain - c * kc : (uint64_t)kc) / 4);
    // 32 columns per step: the 16 shared loads issue together, then the
    // chain runs through them (one exposed load latency per 32 columns)
    int k = 0;
    for (; k + 8 <= n4; k += 8) {
      float4 a[8], b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a[u] = lds4(ra + 16 * (k + u));
        b[u] = lds4(va + 16 * (k + u));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) add4(a[u], b[u]);
    }
    for (; k < n4; ++k) add4(lds4(ra + 16 * k), lds4(va + 16 * k));
    __syncwarp();   // every lane is done with the stage before it is refilled
    issue(c + kSqStages);
  }
  if (lane < nrow) {
    const float* row = A + (r0 + lane) * lda;
    for (uint64_t j = cmain; j < cols; ++j) add(row[j], v[j]);
    y[r0 + lane] = (float)acc;
  }
}

// rows per warp: one chain set per SM sub-partition (148 x 4), at most 32
static int seq_rows_per_warp(uint64_t rows) {
  const uint64_t want = (rows + 148 * kSqWarps - 1) / (148 * kSqWarps);
  return want >= 32 ? 32 : (int)std::max<uint64_t>(want, 1);
}

static bool seq_staged_ok(const float* A, uint64_t lda, const float* v) {
  return ((uintptr_t)A % 16 == 0) && ((uintptr_t)v % 16 == 0) && lda % 4 == 0;
}

// mpgemv.gemv_oracle (mpgemv.py:64-69) on binary64 inputs: binary64
// products, sequential binary64 sum (np.cumsum order); one thread per row.
__global__ void k_gemv_oracle64(const double* A, uint64_t lda, uint64_t rows, uint64_t cols, const double* v,
                                double* y) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const double* row = A + i * lda;
  double acc = 0.0;
  for (uint64_t j = 0; j < cols; ++j) acc = __dadd_rn(acc, __dmul_rn(row[j], v[j]));
  y[i] = acc;
}

// fixed-fanout tree (K:50-77): leaf level from products, groups summed
// left to right, tail padded with zeros.  out is rows x ng.
template <int POL, typename T>
__global__ void k_gemv_tree_leaf(const float* A, uint64_t lda, uint64_t rows, uint64_t cols,
                                 const float* v, int fanout, T* out, uint64_t ng) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= rows * ng) return;
  const uint64_t i = t / ng, g = t % ng;
  const float* row = A + i * lda;
  auto prod = [&](uint64_t j) -> T {
    if (POL == WHFF_POLICY_DOUBLE) return (T)__dmul_rn((double)row[j], (double)ldg(v + j));
    return (T)__fmul_rn(row[j], ldg(v + j));
  };
  const uint64_t j0 = g * (uint64_t)fanout;
  T acc = prod(j0);
  for (int k = 1; k < fanout; ++k) {
    const uint64_t j = j0 + k;
    const T term = j < cols ? prod(j) : (T)0;
    acc = acc + term;
  }
  out[i * ng + g] = acc;
}

template <typename T>
__global__ void k_gemv_tree_level(const T* in, uint64_t rows, uint64_t w, int fanout, T* out,
                                  uint64_t ng) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= rows * ng) return;
  const uint64_t i = t / ng, g = t % ng;
  const T* r = in + i * w;
  const uint64_t j0 = g * (uint64_t)fanout;
  T acc = r[j0];
  for (int k = 1; k < fanout; ++k) {
    const uint64_t j = j0 + k;
    acc = acc + (j < w ? r[j] : (T)0);
  }
  out[i * ng + g] = acc;
}

template <typename T>
__global__ void k_tree_store(const T* in, uint64_t rows, float* y) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < rows) y[i] = (float)in[i];
}

// B200 blocked order: warp per (row, segment of seg_cols columns).  Each lane
// issues kBlkU 16-byte loads of the row (streaming, evict-first) and of the
// vector before using any of them, so a warp keeps kBlkU x 512 B in flight;
// two accumulators per lane (even / odd float4 of the batch) break the add
// chain.  Partials: xor butterfly, then k_blocked_finish adds the segments in
// order.  Deterministic for a given shape.
constexpr int kBlkU = 8;
template <int POL>
__global__ void __launch_bounds__(256) k_gemv_blocked(const float* A, uint64_t lda, uint64_t rows,
                                                      uint64_t cols, const float* v, uint64_t nseg,
                                                      uint64_t seg_cols, bool vec4, double* part) {
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  if (gw >= rows * nseg) return;
  const int lane = threadIdx.x & 31;
  const uint64_t i = gw / nseg, sg = gw % nseg;
  const float* row = A + i * lda;
  const uint64_t c0 = sg * seg_cols;
  const uint64_t c1 = min(cols, c0 + seg_cols);
  double accd[2] = {0.0, 0.0};
  float accf[2] = {0.0f, 0.0f};
  auto add = [&](int k, float a, float b) {
    if (POL == WHFF_POLICY_SINGLE) accf[k] = __fadd_rn(accf[k], __fmul_rn(a, b));
    else if (POL == WHFF_POLICY_MIXED) accd[k] = __dadd_rn(accd[k], (double)__fmul_rn(a, b));
    else accd[k] = __dadd_rn(accd[k], __dmul_rn((double)a, (double)b));
  };
  uint64_t j0 = c0;
  if (vec4) {
    const float4* r4 = reinterpret_cast<const float4*>(row);
    const float4* v4 = reinterpret_cast<const float4*>(v);
    const uint64_t q1 = c1 / 4;
    uint64_t q = c0 / 4;                       // c0 is a multiple of 512 (seg_cols)
    for (; q + 32 * kBlkU <= q1; q += 32 * kBlkU) {
      float4 a[kBlkU], b[kBlkU];
#pragma unroll
      for (int u = 0; u < kBlkU; ++u) {
        a[u] = __ldcs(r4 + q + 32 * u + lane);
        b[u] = ldg(v4 + q + 32 * u + lane);
      }
#pragma unroll
      for (int u = 0; u < kBlkU; ++u) {
        add(u & 1, a[u].x, b[u].x); add(u & 1, a[u].y, b[u].y);
        add(u & 1, a[u].z, b[u].z); add(u & 1, a[u].w, b[u].w);
      }
    }
    for (uint64_t r = q + lane; r < q1; r += 32) {
      const float4 a = __ldcs(r4 + r), b = ldg(v4 + r);
      add(0, a.x, b.x); add(0, a.y, b.y); add(0, a.z, b.z); add(0, a.w, b.w);
    }
    j0 = q1 * 4;
  }
  for (uint64_t j = j0 + lane; j < c1; j += 32) add(0, row[j], ldg(v + j));
  double ad = __dadd_rn(accd[0], accd[1]);
  float af = __fadd_rn(accf[0], accf[1]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ad = __dadd_rn(ad, __shfl_xor_sync(0xFFFFFFFFu, ad, o));
    af = __fadd_rn(af, __shfl_xor_sync(0xFFFFFFFFu, af, o));
  }
  if (lane == 0) part[gw] = POL == WHFF_POLICY_SINGLE ? (double)af : ad;
}

template <int POL>
__global__ void k_blocked_finish(const double* part, uint64_t rows, uint64_t nseg, float* y) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  if (POL == WHFF_POLICY_SINGLE) {
    float acc = 0.0f;
    for (uint64_t s = 0; s < nseg; ++s) acc = __fadd_rn(acc, (float)part[i * nseg + s]);
    y[i] = acc;
  } else {
    double acc = 0.0;
    for (uint64_t s = 0; s < nseg; ++s) acc = __dadd_rn(acc, part[i * nseg + s]);
    y[i] = __double2float_rn(acc);
  }
}

// First non-finite element (mpgemv.py:42-51, codec.py:312-313): grid-stride
// over float4 with four streaming loads in flight per thread; the minimum
// index over threads via atomicMin.
__global__ void k_find_nonfinite(const float* x, uint64_t n, unsigned long long* status) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long bad = ~0ull;
  auto nonfinite = [](float f) { return (__float_as_uint(f) & 0x7F800000u) == 0x7F800000u; };
  uint64_t j0 = 0;
  if ((reinterpret_cast<uintptr_t>(x) & 15u) == 0) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const uint64_t n4 = n / 4;
    for (uint64_t q = tid; q < n4 && bad == ~0ull; q += 4 * nt) {
      float4 a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint64_t k = q + u * nt;
        a[u] = k < n4 ? __ldcs(x4 + k) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float e[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (nonfinite(e[c])) bad = min(bad, (unsigned long long)(4 * (q + u * nt) + c));
      }
    }
    j0 = n4 * 4;
  }
  for (uint64_t i = j0 + tid; i < n && bad == ~0ull; i += nt)
    if (nonfinite(ldg(x + i))) bad = i;
  if (bad != ~0ull) atomicMin(status, bad);
}

// ---------------------------------------------------------------------------
// Thermal (thermal.py:81-117): CSR binary64, CSR order, binary32 store
// ---------------------------------------------------------------------------
__global__ void k_csr_matvec(const int64_t* indptr, const int32_t* indices, const double* data,
                             uint64_t n, const float* x, const float* bdiag, const float* u,
                             float* y) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  const int64_t e = indptr[i + 1];
  // eight entries at a time: their loads and gathers are issued together
  // (two memory round trips per eight instead of two per entry); the sum
  // stays in the row's order (scipy's)
  for (int64_t b = indptr[i]; b < e; b += 8) {
    double d[8];
    float xv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      d[k] = 0.0;
      xv[k] = 0.0f;
      if (b + k < e) {
        d[k] = ldg(data + b + k);
        xv[k] = ldg(x + ldg(indices + b + k));
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (b + k < e) acc = __dadd_rn(acc, __dmul_rn(d[k], (double)xv[k]));
  }
  if (bdiag != nullptr) acc = __dadd_rn(acc, __dmul_rn((double)bdiag[i], (double)u[i]));
  y[i] = __double2float_rn(acc);
}

// device clock for run_scan pacing (pipeline.py:164-289 real-time mode)
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void k_timestamp(uint64_t* t) { *t = globaltimer(); }
__global__ void k_wait_until(const uint64_t* base, uint64_t offset_ns) {
  const uint64_t target = *base + offset_ns;
  while (globaltimer() < target) __nanosleep(2000);
}

__global__ void k_source_term(const float* fp, const float* dark, float dose, uint64_t n, float* u) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  u[i] = fp ? __fadd_rn(__fmul_rn(dose, fp[i]), dark[i]) : dark[i];
}

// ---------------------------------------------------------------------------
// skeleton-first layout (whff_relayout.cuh): per-block permutation
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_relayout(StreamView s, const uint32_t* in, uint32_t* out,
                                                  int inverse) {
  const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (b >= s.br * s.bc) return;
  uint64_t start;
  int len;
  block_extent(s, b, start, len);
  if (inverse) unrelayout_segment(in, out, start, len, s.planes_limit, s.has_raw != 0);
  else relayout_segment(in, out, start, len, s.planes_limit, s.has_raw != 0);
}

// ---------------------------------------------------------------------------
// GPU encoder (codec.py:225-293, K:139-283)
// ---------------------------------------------------------------------------
// One thread per block, a long dependent chain (transform, plane search,
// bit-plane emission) and little memory traffic: occupancy hides it, so both
// passes are held to 64 registers (8 CTAs of 128 per SM).  Paper slit
// (378 x 256,000): FixedRate(8) 10.4 -> 5.6 ms (also: no counting pass at a
// fixed rate), FixedAccuracy(1e-12) 7.1 -> 6.0 ms, FixedPrecision(17) 6.1 ->
// 4.5 ms; byte-identical streams (scratch sweep of 1, 6, 8 CTAs per SM).
#ifndef WHFF_ENC_MINB
#define WHFF_ENC_MINB 8
#endif
__global__ void __launch_bounds__(128, WHFF_ENC_MINB) k_encode_len(const float* a, uint64_t lda, uint64_t rows,
                                                                  uint64_t cols, uint64_t nb, uint64_t bc, int mode,
                                                                  double param, uint64_t* lens, int* overflow) {
  const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (b >= nb) return;
  BlockPlan pl;
  plan_block(a, (int64_t)lda, (int64_t)rows, (int64_t)cols, (int64_t)b, (int64_t)bc, mode, param, pl);
  if (!pl.ok) atomicOr(overflow, 1);
  const int budget = mode == WHFF_MODE_RATE ? (int)param * 16 : 0;
  // FixedRate: every block takes exactly its budget (codec.py:268-272, the
  // stream pads short blocks), so there is nothing to count
  int n = budget;
  if (!budget) {
    CountSink cs;
    n = encode_one(pl.mag, pl.negm, pl.code, pl.planes, pl.raw, pl.raw_words, 0, mode == WHFF_MODE_ACCURACY, cs);
  }
  lens[b] = (uint64_t)n;
}

__global__ void __launch_bounds__(128, WHFF_ENC_MINB) k_encode_emit(const float* a, uint64_t lda, uint64_t rows, uint64_t cols, uint64_t nb,
                              uint64_t bc, int mode, double param, const uint64_t* offsets,
                              uint32_t* words) {
  const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (b >= nb) return;
  BlockPlan pl;
  plan_block(a, (int64_t)lda, (int64_t)rows, (int64_t)cols, (int64_t)b, (int64_t)bc, mode, param, pl);
  const int budget = mode == WHFF_MODE_RATE ? (int)param * 16 : 0;
  WordSink ws{words, offsets[b], 0u, 0, budget ? budget : 0x7FFFFFFF};
  encode_one(pl.mag, pl.negm, pl.code, pl.planes, pl.raw, pl.raw_words, budget,
             mode == WHFF_MODE_ACCURACY, ws);
  ws.finish();
}

struct EncArrays {
  const uint32_t* mag;
  const uint8_t* neg;
  const uint16_t* emax;
  const uint8_t* planes;
  const uint8_t* raw_mask;
  const uint32_t* raw_words;
};

__device__ void load_enc(const EncArrays& E, uint64_t b, int has_raw, uint32_t mag[16],
                         uint32_t& negm, uint32_t& code, int& planes, bool& raw, uint32_t rw[16]) {
  negm = 0;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    mag[c] = E.mag[16 * b + c];
    if (E.neg[16 * b + c]) negm |= 1u << c;
    rw[c] = E.raw_words[16 * b + c];
  }
  code = E.emax[b];
  planes = E.planes[b];
  raw = has_raw && E.raw_mask[b];
}

__global__ void k_encblocks_len(EncArrays E, uint64_t nb, int budget, int has_raw, uint64_t* lens) {
  const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (b >= nb) return;
  uint32_t mag[16], rw[16], negm, code;
  int planes;
  bool raw;
  load_enc(E, b, has_raw, mag, negm, code, planes, raw, rw);
  CountSink cs;
  int n = encode_one(mag, negm, code, planes, raw, rw, budget, has_raw != 0, cs);
  if (budget) n = budget;
  lens[b] = (uint64_t)n;
}

__global__ void k_encblocks_emit(EncArrays E, uint64_t nb, int budget, int has_raw,
                                 const uint64_t* offsets, uint32_t* words) {
  const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (b >= nb) return;
  uint32_t mag[16], rw[16], negm, code;
  int planes;
  bool raw;
  load_enc(E, b, has_raw, mag, negm, code, planes, raw, rw);
  WordSink ws{words, offsets[b], 0u, 0, budget ? budget : 0x7FFFFFFF};
  encode_one(mag, negm, code, planes, raw, rw, budget, has_raw != 0, ws);
  ws.finish();
}

// compact index from u64 offsets (device-encoded streams)
__global__ void k_build_compact(const uint64_t* offsets, uint64_t nb, uint64_t bc, uint64_t gpr,
                                uint64_t payload_bits, uint16_t* lens, uint64_t* base) {
  const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const uint64_t s = offsets[b];
  const uint64_t e = b + 1 < nb ? offsets[b + 1] : payload_bits;
  const uint64_t l = e > s ? e - s : 0;
  lens[b] = (uint16_t)(l > 65535 ? 65535 : l);
  const uint64_t brow = b / bc, bcol = b % bc;
  if ((bcol & 31) == 0) base[brow * gpr + (bcol >> 5)] = s;
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
namespace {

inline unsigned grid_for(uint64_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }

// the per-launch vector prologue: U = G^T v (coefficient) or padded v (exact
// evaluation of a packed stream)
static void vec_prologue(int eval, const float* v, uint64_t cols, uint64_t bc, float4* out, cudaStream_t cs) {
  if (eval == WHFF_EVAL_COEFF)
    k_coeff_prep<<<grid_for(pad_tiles(bc), 256), 256, 0, cs>>>(v, cols, bc, pad_tiles(bc), out);
  else
    k_vpad<<<grid_for(pad_tiles(bc), 256), 256, 0, cs>>>(v, cols, bc, pad_tiles(bc), out);
}


struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int planes_limit_for(int mode, double param) {
  if (mode == WHFF_MODE_PRECISION) {
    const int p = (int)param;
    return p < kNPlanes ? p : kNPlanes;
  }
  return kNPlanes;
}

whff_status_t check_mode(int mode, double param) {
  if (mode == WHFF_MODE_RATE) {
    if (!(param >= 1 && param <= 32 && param == (double)(int)param))
      return fail(WHFF_ERR_ARGUMENT, "fixed-rate bits per value must be in 1..32");
  } else if (mode == WHFF_MODE_PRECISION) {
    if (!(param >= 1 && param <= 32 && param == (double)(int)param))
      return fail(WHFF_ERR_ARGUMENT, "fixed-precision planes must be in 1..32");
  } else if (mode == WHFF_MODE_ACCURACY) {
    if (!(param >= 0.0)) return fail(WHFF_ERR_ARGUMENT, "tolerance must be nonnegative");
  } else {
    return fail(WHFF_ERR_ARGUMENT, "unknown codec mode");
  }
  return WHFF_OK;
}

whff_status_t alloc_payload(whff_dstream* s, uint64_t bytes) {
  s->payload_alloc = ((bytes + 15) / 16) * 16 + 64;  // >= 32 readable pad bytes
  WCK(cudaMalloc(&s->d_payload, s->payload_alloc));
  WCK(cudaMemset(s->d_payload, 0, s->payload_alloc));
  return WHFF_OK;
}

void free_stream(whff_dstream* s) {
  if (!s) return;
  DeviceGuard g(s->device);
  cudaFree(s->d_payload);
  cudaFree(s->d_base);
  cudaFree(s->d_lens);
  cudaFree(s->d_starts);
  cudaFree(s->d_pk_body);
  cudaFree(s->d_pk_segs);
  cudaFree(s->d_pk_exc_block);
  cudaFree(s->d_pk_exc_words);
  delete s;
}

void drop_packed(whff_dstream* s) {
  if (!s->packed) return;
  DeviceGuard g(s->device);
  cudaFree(s->d_pk_body);
  cudaFree(s->d_pk_segs);
  cudaFree(s->d_pk_exc_block);
  cudaFree(s->d_pk_exc_words);
  s->d_pk_body = nullptr;
  s->d_pk_segs = nullptr;
  s->d_pk_exc_block = nullptr;
  s->d_pk_exc_words = nullptr;
  s->packed = false;
  s->pk_body_words = s->pk_nexc = s->pk_alloc_words = 0;
  s->pk_band_bytes.clear();
}

PkView pk_view(const whff_dstream* s) {
  PkView v;
  v.g = pk::make_geom(s->rows, s->cols, pk::seg_tiles_for_mode(s->mode));
  v.body = s->d_pk_body;
  v.segs = s->d_pk_segs;
  v.pars = s->d_pk_segs ? reinterpret_cast<const pk::FieldPar*>(s->d_pk_segs + v.g.nband * v.g.nsegb) : nullptr;
  v.exc_block = s->d_pk_exc_block;
  v.exc_words = s->d_pk_exc_words;
  return v;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

int whff_abi_version(void) { return WHFF_ABI_VERSION; }

const char* whff_status_string(whff_status_t s) {
  switch (s) {
    case WHFF_OK: return "ok";
    case WHFF_ERR_DIMENSION: return "dimension error";
    case WHFF_ERR_NONFINITE: return "non-finite value";
    case WHFF_ERR_CORRUPT: return "corrupt stream";
    case WHFF_ERR_ARGUMENT: return "invalid argument";
    case WHFF_ERR_OVERFLOW: return "internal error: transform coefficient overflow";
    case WHFF_ERR_NOMEM: return "out of memory";
    case WHFF_ERR_CUDA: return "cuda error";
  }
  return "unknown";
}

const char* whff_last_error(void) { return g_err.c_str(); }

whff_status_t whff_dstream_create(int device, int mode, double param, uint64_t rows, uint64_t cols,
                                  const uint8_t* payload, uint64_t payload_bytes,
                                  const uint64_t* index, uint64_t nb, whff_dstream_t* out) {
  if (!out) return fail(WHFF_ERR_ARGUMENT, "null output handle");
  *out = nullptr;
  whff_status_t st = check_mode(mode, param);
  if (st != WHFF_OK) return st;
  if (rows < 1 || cols < 1) return fail(WHFF_ERR_DIMENSION, "stream dimensions must be positive");
  const uint64_t br = (rows + 3) / 4, bc = (cols + 3) / 4;
  // codec.py:347-356 _validate_stream
  if (nb != br * bc) return fail(WHFF_ERR_CORRUPT, "block index length does not match dimensions");
  if (payload_bytes > 0 && !payload) return fail(WHFF_ERR_ARGUMENT, "null payload");
  if (!index) return fail(WHFF_ERR_ARGUMENT, "null block index");
  const uint64_t pbits = payload_bytes * 8;
  uint64_t mx = 0;
  for (uint64_t b = 0; b < nb; ++b) mx = index[b] > mx ? index[b] : mx;
  if (mx >= std::max<uint64_t>(pbits, 1))
    return fail(WHFF_ERR_CORRUPT, "block index offsets point past the payload");
  // codec.py:335-344 _segment_lengths (variable modes)
  if (mode != WHFF_MODE_RATE) {
    for (uint64_t b = 0; b + 1 < nb; ++b)
      if (index[b + 1] < index[b])
        return fail(WHFF_ERR_CORRUPT, "block index offsets are not nondecreasing");
  }
  DeviceGuard g(device);
  whff_dstream* s = new whff_dstream();
  s->device = device;
  s->mode = mode;
  s->param = param;
  s->rows = rows;
  s->cols = cols;
  s->br = br;
  s->bc = bc;
  s->nb = nb;
  s->gpr = (bc + 31) / 32;
  s->payload_bytes = payload_bytes;
  s->payload_bits = pbits;
  s->planes_limit = planes_limit_for(mode, param);
  s->has_raw = mode == WHFF_MODE_ACCURACY;
  s->seg_bits = mode == WHFF_MODE_RATE ? (uint32_t)param * 16u : 0u;
  st = alloc_payload(s, payload_bytes);
  if (st != WHFF_OK) { free_stream(s); return st; }
  if (payload_bytes) {
    cudaError_t e = cudaMemcpy(s->d_payload, payload, payload_bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { free_stream(s); return cuda_fail(e, "upload payload"); }
  }
  // choose the index layout
  bool implicit = mode == WHFF_MODE_RATE;
  for (uint64_t b = 0; implicit && b < nb; ++b) implicit = index[b] == b * s->seg_bits;
  std::vector<uint16_t> lens;
  if (implicit) {
    s->kind = WHFF_INDEX_IMPLICIT;
  } else {
    lens.resize(nb);
    bool compact = mode != WHFF_MODE_RATE;
    for (uint64_t b = 0; b < nb; ++b) {
      uint64_t l;
      if (mode == WHFF_MODE_RATE) {
        l = s->seg_bits;
      } else {
        const uint64_t e = b + 1 < nb ? index[b + 1] : pbits;
        l = e - index[b];
        if (b + 1 < nb && l > 65535) compact = false;
      }
      lens[b] = (uint16_t)(l > 65535 ? 65535 : l);
    }
    s->kind = compact ? WHFF_INDEX_COMPACT : WHFF_INDEX_FULL;
    cudaError_t e = cudaMalloc(&s->d_lens, nb * sizeof(uint16_t));
    if (e == cudaSuccess) e = cudaMemcpy(s->d_lens, lens.data(), nb * 2, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
      if (compact) {
        std::vector<uint64_t> base(br * s->gpr);
        for (uint64_t r = 0; r < br; ++r)
          for (uint64_t gg = 0; gg < s->gpr; ++gg) base[r * s->gpr + gg] = index[r * bc + gg * 32];
        e = cudaMalloc(&s->d_base, base.size() * 8);
        if (e == cudaSuccess) e = cudaMemcpy(s->d_base, base.data(), base.size() * 8, cudaMemcpyHostToDevice);
        s->index_bytes = nb * 2 + base.size() * 8;
      } else {
        e = cudaMalloc(&s->d_starts, nb * 8);
        if (e == cudaSuccess) e = cudaMemcpy(s->d_starts, index, nb * 8, cudaMemcpyHostToDevice);
        s->index_bytes = nb * 10;
      }
    }
    if (e != cudaSuccess) { free_stream(s); return cuda_fail(e, "upload index"); }
  }
  *out = s;
  return WHFF_OK;
}

whff_status_t whff_dstream_create_segments(int device, const uint8_t* payload, uint64_t payload_bytes,
                                           const uint64_t* offsets, const uint64_t* seglens, uint64_t nb,
                                           int planes_limit, int has_raw, whff_dstream_t* out) {
  if (!out) return fail(WHFF_ERR_ARGUMENT, "null output handle");
  *out = nullptr;
  if (nb == 0) return fail(WHFF_ERR_DIMENSION, "empty segment table");
  if ((payload_bytes && !payload) || !offsets || !seglens) return fail(WHFF_ERR_ARGUMENT, "null argument");
  DeviceGuard g(device);
  whff_dstream* s = new whff_dstream();
  s->device = device;
  s->mode = has_raw ? WHFF_MODE_ACCURACY : WHFF_MODE_PRECISION;
  s->param = planes_limit;
  s->rows = 4;
  s->cols = 4 * nb;
  s->br = 1;
  s->bc = nb;
  s->nb = nb;
  s->gpr = (nb + 31) / 32;
  s->payload_bytes = payload_bytes;
  s->payload_bits = payload_bytes * 8;
  s->planes_limit = planes_limit < 0 ? kNPlanes : std::min(planes_limit, kNPlanes);
  s->has_raw = has_raw != 0;
  s->seg_bits = 0;
  s->kind = WHFF_INDEX_FULL;
  whff_status_t st = alloc_payload(s, payload_bytes);
  if (st != WHFF_OK) { free_stream(s); return st; }
  std::vector<uint16_t> lens(nb);
  for (uint64_t b = 0; b < nb; ++b) lens[b] = (uint16_t)std::min<uint64_t>(seglens[b], 65535);
  cudaError_t e = payload_bytes ? cudaMemcpy(s->d_payload, payload, payload_bytes, cudaMemcpyHostToDevice)
                                : cudaSuccess;
  if (e == cudaSuccess) e = cudaMalloc(&s->d_lens, nb * 2);
  if (e == cudaSuccess) e = cudaMemcpy(s->d_lens, lens.data(), nb * 2, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&s->d_starts, nb * 8);
  if (e == cudaSuccess) e = cudaMemcpy(s->d_starts, offsets, nb * 8, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { free_stream(s); return cuda_fail(e, "segment stream upload"); }
  s->index_bytes = nb * 10;
  *out = s;
  return WHFF_OK;
}

// permuted copy of the payload (forward: reference -> skeleton-first)
static whff_status_t permuted_payload(const whff_dstream* s, bool inverse, uint8_t** out,
                                      cudaStream_t cs) {
  uint8_t* np = nullptr;
  cudaError_t e = cudaMalloc(&np, s->payload_alloc);
  if (e == cudaSuccess) e = cudaMemcpyAsync(np, s->d_payload, s->payload_alloc, cudaMemcpyDeviceToDevice, cs);
  if (e != cudaSuccess) { cudaFree(np); return cuda_fail(e, "relayout alloc"); }
  StreamView v = s->view();
  k_relayout<<<grid_for(s->nb, 128), 128, 0, cs>>>(v, reinterpret_cast<const uint32_t*>(s->d_payload),
                                                    reinterpret_cast<uint32_t*>(np), inverse ? 1 : 0);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) { cudaFree(np); return cuda_fail(e, "relayout"); }
  *out = np;
  return WHFF_OK;
}

whff_status_t whff_dstream_relayout(whff_dstream_t s, int layout, whff_stream_t stream) {
  if (!s) return fail(WHFF_ERR_ARGUMENT, "null stream");
  if (layout != WHFF_LAYOUT_REFERENCE && layout != WHFF_LAYOUT_SKELETON_FIRST)
    return fail(WHFF_ERR_ARGUMENT, "unknown layout");
  if (layout == s->layout) return WHFF_OK;
  if (s->kind == WHFF_INDEX_FULL)
    return fail(WHFF_ERR_ARGUMENT, "relayout needs an implicit or compact index");
  DeviceGuard g(s->device);
  uint8_t* np = nullptr;
  whff_status_t st = permuted_payload(s, layout == WHFF_LAYOUT_REFERENCE, &np, (cudaStream_t)stream);
  if (st != WHFF_OK) return st;
  cudaFree(s->d_payload);
  s->d_payload = np;
  s->layout = layout;
  return WHFF_OK;
}

// Build the tile-packed representation (whff_packed.cuh) from the stream's
// payload: pass 1 sizes every segment, two scans place them, pass 2 writes
// records and exceptions.  Synchronous on `stream`.
whff_status_t whff_dstream_pack(whff_dstream_t s, whff_stream_t stream) {
  if (!s) return fail(WHFF_ERR_ARGUMENT, "null stream");
  if (s->packed) return WHFF_OK;
  DeviceGuard g(s->device);
  cudaStream_t cs = (cudaStream_t)stream;
  const pk::Geom gg = pk::make_geom(s->rows, s->cols, pk::seg_tiles_for_mode(s->mode));
  const uint64_t nseg = gg.nband * gg.nsegb;
  pk::Seg* segs = nullptr;
  uint64_t *words = nullptr, *exc = nullptr, *off = nullptr, *eoff = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0, t2 = 0;
  cudaError_t e = cudaMalloc(&segs, pk_segs_bytes(nseg));
  if (e == cudaSuccess) e = cudaMalloc(&words, (nseg + 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&exc, (nseg + 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&off, (nseg + 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&eoff, (nseg + 1) * 8);
  if (e == cudaSuccess) e = cudaMemsetAsync(words + nseg, 0, 8, cs);
  if (e == cudaSuccess) e = cudaMemsetAsync(exc + nseg, 0, 8, cs);
  auto cleanup = [&]() {
    cudaFree(words);
    cudaFree(exc);
    cudaFree(off);
    cudaFree(eoff);
    cudaFree(tmp);
  };
  if (e != cudaSuccess) { cleanup(); cudaFree(segs); return cuda_fail(e, "pack alloc"); }
  const StreamView v = s->view();
  e = pk_launch_stats(v, gg, segs, words, exc, cs);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, words, off, (int)(nseg + 1), cs);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(nullptr, t2, exc, eoff, (int)(nseg + 1), cs);
  tmp_bytes = std::max(tmp_bytes, t2);
  if (e == cudaSuccess) e = cudaMalloc(&tmp, tmp_bytes);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, words, off, (int)(nseg + 1), cs);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, exc, eoff, (int)(nseg + 1), cs);
  uint64_t tot[2] = {0, 0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(&tot[0], off + nseg, 8, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&tot[1], eoff + nseg, 8, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e == cudaSuccess) e = pk_launch_finalize(segs, nseg, off, eoff, cs);
  if (e == cudaSuccess) e = pk_launch_params(segs, nseg, cs);
  // readable slack past the body: rows past a band's end and tails read ahead
  const uint64_t alloc_words = tot[0] + 4 * pk::kMaxRecordWords * 32 + 64;
  uint32_t* body = nullptr;
  uint64_t* xb = nullptr;
  uint32_t* xw = nullptr;
  const uint64_t ne = std::max<uint64_t>(tot[1], 1);
  if (e == cudaSuccess) e = cudaMalloc(&body, alloc_words * 4);
  if (e == cudaSuccess) e = cudaMemsetAsync(body, 0, alloc_words * 4, cs);
  if (e == cudaSuccess) e = cudaMalloc(&xb, ne * 8);
  if (e == cudaSuccess) e = cudaMalloc(&xw, ne * 64);
  if (e == cudaSuccess) e = pk_launch_emit(v, gg, segs, body, xb, xw, cs);
  std::vector<uint64_t> hoff(nseg + 1), hexc(nseg + 1);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hoff.data(), off, (nseg + 1) * 8, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hexc.data(), eoff, (nseg + 1) * 8, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  cleanup();
  if (e != cudaSuccess) {
    cudaFree(segs);
    cudaFree(body);
    cudaFree(xb);
    cudaFree(xw);
    return cuda_fail(e, "pack");
  }
  s->d_pk_body = body;
  s->d_pk_segs = segs;
  s->d_pk_exc_block = xb;
  s->d_pk_exc_words = xw;
  s->pk_body_words = tot[0];
  s->pk_nexc = tot[1];
  s->pk_alloc_words = alloc_words;
  s->pk_band_bytes.assign(gg.nband, 0);
  for (uint64_t b = 0; b < gg.nband; ++b) {
    const uint64_t s0 = b * gg.nsegb, s1 = s0 + gg.nsegb;
    s->pk_band_bytes[b] = (hoff[s1] - hoff[s0]) * 4 + gg.nsegb * (sizeof(pk::Seg) + 16 * sizeof(pk::FieldPar)) +
                          (hexc[s1] - hexc[s0]) * 72;
  }
  s->packed = true;
  return WHFF_OK;
}

whff_status_t whff_dstream_packed_download(whff_dstream_t s, uint8_t* segs, uint32_t* body, uint64_t* xb,
                                           uint32_t* xw, uint64_t* n_segs, uint64_t* body_words,
                                           uint64_t* n_exc) {
  if (!s) return fail(WHFF_ERR_ARGUMENT, "null stream");
  if (!s->packed) return fail(WHFF_ERR_ARGUMENT, "stream is not packed (whff_dstream_pack)");
  const pk::Geom gg = pk::make_geom(s->rows, s->cols, pk::seg_tiles_for_mode(s->mode));
  const uint64_t nseg = gg.nband * gg.nsegb;
  if (n_segs) *n_segs = nseg;
  if (body_words) *body_words = s->pk_body_words;
  if (n_exc) *n_exc = s->pk_nexc;
  DeviceGuard g(s->device);
  if (segs) WCK(cudaMemcpy(segs, s->d_pk_segs, nseg * sizeof(pk::Seg), cudaMemcpyDeviceToHost));
  if (body && s->pk_body_words) WCK(cudaMemcpy(body, s->d_pk_body, s->pk_body_words * 4, cudaMemcpyDeviceToHost));
  if (xb && s->pk_nexc) WCK(cudaMemcpy(xb, s->d_pk_exc_block, s->pk_nexc * 8, cudaMemcpyDeviceToHost));
  if (xw && s->pk_nexc) WCK(cudaMemcpy(xw, s->d_pk_exc_words, s->pk_nexc * 64, cudaMemcpyDeviceToHost));
  return WHFF_OK;
}

whff_status_t whff_dstream_clone(whff_dstream_t s, whff_dstream_t* out) {
  if (!s || !out) return fail(WHFF_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  DeviceGuard g(s->device);
  whff_dstream* c = new whff_dstream(*s);
  c->d_payload = nullptr;
  c->d_base = nullptr;
  c->d_lens = nullptr;
  c->d_starts = nullptr;
  c->d_pk_body = nullptr;
  c->d_pk_segs = nullptr;
  c->d_pk_exc_block = nullptr;
  c->d_pk_exc_words = nullptr;
  cudaError_t e = cudaMalloc(&c->d_payload, s->payload_alloc);
  if (e == cudaSuccess) e = cudaMemcpy(c->d_payload, s->d_payload, s->payload_alloc, cudaMemcpyDeviceToDevice);
  if (e == cudaSuccess && s->d_base) {
    e = cudaMalloc(&c->d_base, s->br * s->gpr * 8);
    if (e == cudaSuccess) e = cudaMemcpy(c->d_base, s->d_base, s->br * s->gpr * 8, cudaMemcpyDeviceToDevice);
  }
  if (e == cudaSuccess && s->d_lens) {
    e = cudaMalloc(&c->d_lens, s->nb * 2);
    if (e == cudaSuccess) e = cudaMemcpy(c->d_lens, s->d_lens, s->nb * 2, cudaMemcpyDeviceToDevice);
  }
  if (e == cudaSuccess && s->d_starts) {
    e = cudaMalloc(&c->d_starts, s->nb * 8);
    if (e == cudaSuccess) e = cudaMemcpy(c->d_starts, s->d_starts, s->nb * 8, cudaMemcpyDeviceToDevice);
  }
  if (e == cudaSuccess && s->packed) {
    const pk::Geom gg = pk::make_geom(s->rows, s->cols, pk::seg_tiles_for_mode(s->mode));
    const uint64_t nseg = gg.nband * gg.nsegb;
    e = cudaMalloc(&c->d_pk_body, s->pk_alloc_words * 4);
    if (e == cudaSuccess)
      e = cudaMemcpy(c->d_pk_body, s->d_pk_body, s->pk_alloc_words * 4, cudaMemcpyDeviceToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_pk_segs, pk_segs_bytes(nseg));
    if (e == cudaSuccess)
      e = cudaMemcpy(c->d_pk_segs, s->d_pk_segs, pk_segs_bytes(nseg), cudaMemcpyDeviceToDevice);
    const uint64_t ne = std::max<uint64_t>(s->pk_nexc, 1);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_pk_exc_block, ne * 8);
    // (the exception list has a placeholder entry when empty: copy the real ones)
    if (e == cudaSuccess && s->pk_nexc)
      e = cudaMemcpy(c->d_pk_exc_block, s->d_pk_exc_block, s->pk_nexc * 8, cudaMemcpyDeviceToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_pk_exc_words, ne * 64);
    if (e == cudaSuccess && s->pk_nexc)
      e = cudaMemcpy(c->d_pk_exc_words, s->d_pk_exc_words, s->pk_nexc * 64, cudaMemcpyDeviceToDevice);
  }
  if (e != cudaSuccess) { free_stream(c); return cuda_fail(e, "clone"); }
  *out = c;
  return WHFF_OK;
}

whff_status_t whff_dstream_destroy(whff_dstream_t s) {
  free_stream(s);
  return WHFF_OK;
}

whff_status_t whff_dstream_get_info(whff_dstream_t s, whff_dstream_info_t* info) {
  if (!s || !info) return fail(WHFF_ERR_ARGUMENT, "null argument");
  info->mode = s->mode;
  info->index_kind = s->kind;
  info->param = s->param;
  info->rows = s->rows;
  info->cols = s->cols;
  info->n_blocks = s->nb;
  info->payload_bytes = s->payload_bytes;
  info->total_bits = s->total_bits ? s->total_bits : s->payload_bits;
  info->index_bytes = s->index_bytes;
  info->device_bytes = s->payload_alloc + s->index_bytes;
  info->planes_limit = s->planes_limit;
  info->has_raw_flag = s->has_raw;
  info->layout = s->layout;
  info->packed = s->packed ? 1 : 0;
  info->device = s->device;
  info->packed_exceptions = s->pk_nexc;
  if (s->packed) {
    const pk::Geom gg = pk::make_geom(s->rows, s->cols, pk::seg_tiles_for_mode(s->mode));
    info->packed_bytes = s->pk_body_words * 4 + pk_segs_bytes(gg.nband * gg.nsegb) + s->pk_nexc * 72;
    info->device_bytes += s->pk_alloc_words * 4 + pk_segs_bytes(gg.nband * gg.nsegb) +
                          std::max<uint64_t>(s->pk_nexc, 1) * 72;
  } else {
    info->packed_bytes = 0;
  }
  return WHFF_OK;
}

whff_status_t whff_dstream_block_row_bits(whff_dstream_t s, uint64_t* out) {
  if (!s || !out) return fail(WHFF_ERR_ARGUMENT, "null argument");
  DeviceGuard g(s->device);
  out[s->br] = s->payload_bits;
  if (s->kind == WHFF_INDEX_IMPLICIT) {
    for (uint64_t b = 0; b < s->br; ++b) out[b] = std::min<uint64_t>(b * s->bc * s->seg_bits, s->payload_bits);
    return WHFF_OK;
  }
  // compact: base[b * gpr] is block (b, 0); full: starts[b * bc]
  const uint64_t* src = s->kind == WHFF_INDEX_COMPACT ? s->d_base : s->d_starts;
  const uint64_t pitch = (s->kind == WHFF_INDEX_COMPACT ? s->gpr : s->bc) * sizeof(uint64_t);
  cudaError_t e = cudaMemcpy2D(out, sizeof(uint64_t), src, pitch, sizeof(uint64_t), s->br, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "block_row_bits");
  return WHFF_OK;
}

// index arrays of a stream as one blob: compact = base (br*gpr u64) + lens
// (nb u16); full = starts (nb u64) + lens (nb u16); implicit = nothing
static uint64_t index_blob_bytes(const whff_dstream* s) {
  if (s->kind == WHFF_INDEX_COMPACT) return s->br * s->gpr * 8 + s->nb * 2;
  if (s->kind == WHFF_INDEX_FULL) return s->nb * 8 + s->nb * 2;
  return 0;
}

whff_status_t whff_dstream_export(whff_dstream_t s, uint8_t* payload, uint64_t* payload_bytes,
                                  uint8_t* index, uint64_t* index_bytes) {
  if (!s) return fail(WHFF_ERR_ARGUMENT, "null stream");
  if (payload_bytes) *payload_bytes = s->payload_bytes;
  if (index_bytes) *index_bytes = index_blob_bytes(s);
  DeviceGuard g(s->device);
  if (payload && s->payload_bytes)
    WCK(cudaMemcpy(payload, s->d_payload, s->payload_bytes, cudaMemcpyDeviceToHost));
  if (index && s->kind != WHFF_INDEX_IMPLICIT) {
    const uint64_t first = s->kind == WHFF_INDEX_COMPACT ? s->br * s->gpr * 8 : s->nb * 8;
    WCK(cudaMemcpy(index, s->kind == WHFF_INDEX_COMPACT ? (const void*)s->d_base : (const void*)s->d_starts,
                   first, cudaMemcpyDeviceToHost));
    WCK(cudaMemcpy(index + first, s->d_lens, s->nb * 2, cudaMemcpyDeviceToHost));
  }
  return WHFF_OK;
}

whff_status_t whff_dstream_reserve(whff_dstream_t s, uint64_t payload_capacity) {
  if (!s) return fail(WHFF_ERR_ARGUMENT, "null stream");
  const size_t want = ((payload_capacity + 15) / 16) * 16 + 64;
  if (want <= s->payload_alloc) return WHFF_OK;
  DeviceGuard g(s->device);
  uint8_t* np = nullptr;
  WCK(cudaMalloc(&np, want));
  cudaError_t e = cudaMemset(np, 0, want);
  if (e == cudaSuccess) e = cudaMemcpy(np, s->d_payload, s->payload_bytes, cudaMemcpyDeviceToDevice);
  if (e != cudaSuccess) { cudaFree(np); return cuda_fail(e, "reserve payload"); }
  cudaFree(s->d_payload);
  s->d_payload = np;
  s->payload_alloc = want;
  return WHFF_OK;
}

whff_status_t whff_dstream_rebind(whff_dstream_t s, uint64_t payload_bytes) {
  if (!s) return fail(WHFF_ERR_ARGUMENT, "null stream");
  if (((payload_bytes + 15) / 16) * 16 + 64 > s->payload_alloc)
    return fail(WHFF_ERR_DIMENSION, "payload exceeds the stream's capacity (whff_dstream_reserve)");
  if (s->kind == WHFF_INDEX_IMPLICIT && payload_bytes != s->payload_bytes)
    return fail(WHFF_ERR_DIMENSION, "fixed-rate payload size differs from the stream's geometry");
  s->payload_bytes = payload_bytes;
  s->payload_bits = payload_bytes * 8;
  if (s->kind != WHFF_INDEX_IMPLICIT) s->total_bits = s->payload_bits;
  drop_packed(s);   // new contents: the packed copy is stale (re-pack to use it)
  return WHFF_OK;
}

whff_status_t whff_dstream_import_async(whff_dstream_t s, const uint8_t* payload, uint64_t payload_bytes,
                                        const uint8_t* index, uint64_t index_bytes, whff_stream_t stream) {
  if (!s || (payload_bytes && !payload)) return fail(WHFF_ERR_ARGUMENT, "null argument");
  if (index_bytes != index_blob_bytes(s))
    return fail(WHFF_ERR_DIMENSION, "imported index does not match the stream's geometry");
  if (index_bytes && !index) return fail(WHFF_ERR_ARGUMENT, "null index");
  // geometry first (host fields: plans created from now on see it) ...
  whff_status_t st = whff_dstream_rebind(s, payload_bytes);
  if (st != WHFF_OK) return st;
  DeviceGuard g(s->device);
  cudaStream_t cs = (cudaStream_t)stream;
  // ... then the bytes, in stream order
  if (payload_bytes) WCK(cudaMemcpyAsync(s->d_payload, payload, payload_bytes, cudaMemcpyHostToDevice, cs));
  if (index_bytes) {
    const uint64_t first = s->kind == WHFF_INDEX_COMPACT ? s->br * s->gpr * 8 : s->nb * 8;
    WCK(cudaMemcpyAsync(s->kind == WHFF_INDEX_COMPACT ? (void*)s->d_base : (void*)s->d_starts, index, first,
                        cudaMemcpyHostToDevice, cs));
    WCK(cudaMemcpyAsync(s->d_lens, index + first, s->nb * 2, cudaMemcpyHostToDevice, cs));
  }
  return WHFF_OK;
}

whff_status_t whff_dstream_download(whff_dstream_t s, uint8_t* payload, uint64_t* index) {
  if (!s) return fail(WHFF_ERR_ARGUMENT, "null stream");
  DeviceGuard g(s->device);
  if (payload && s->payload_bytes) {
    if (s->layout == WHFF_LAYOUT_SKELETON_FIRST) {     // restore the reference bytes
      uint8_t* tmp = nullptr;
      whff_status_t st = permuted_payload(s, true, &tmp, (cudaStream_t)0);
      if (st != WHFF_OK) return st;
      cudaError_t e = cudaMemcpy(payload, tmp, s->payload_bytes, cudaMemcpyDeviceToHost);
      cudaFree(tmp);
      if (e != cudaSuccess) return cuda_fail(e, "download payload");
    } else {
      WCK(cudaMemcpy(payload, s->d_payload, s->payload_bytes, cudaMemcpyDeviceToHost));
    }
  }
  if (index) {
    if (s->kind == WHFF_INDEX_IMPLICIT) {
      for (uint64_t b = 0; b < s->nb; ++b) index[b] = b * s->seg_bits;
    } else if (s->kind == WHFF_INDEX_FULL) {
      WCK(cudaMemcpy(index, s->d_starts, s->nb * 8, cudaMemcpyDeviceToHost));
    } else {
      std::vector<uint16_t> lens(s->nb);
      std::vector<uint64_t> base(s->br * s->gpr);
      WCK(cudaMemcpy(lens.data(), s->d_lens, s->nb * 2, cudaMemcpyDeviceToHost));
      WCK(cudaMemcpy(base.data(), s->d_base, base.size() * 8, cudaMemcpyDeviceToHost));
      for (uint64_t r = 0; r < s->br; ++r) {
        for (uint64_t gg = 0; gg < s->gpr; ++gg) {
          uint64_t st = base[r * s->gpr + gg];
          for (uint64_t c = gg * 32; c < std::min<uint64_t>(s->bc, gg * 32 + 32); ++c) {
            index[r * s->bc + c] = st;
            st += lens[r * s->bc + c];
          }
        }
      }
    }
  }
  return WHFF_OK;
}

whff_status_t whff_compress(const float* a, uint64_t lda, uint64_t rows, uint64_t cols, int mode,
                            double param, whff_stream_t stream, whff_dstream_t* out) {
  if (!out) return fail(WHFF_ERR_ARGUMENT, "null output handle");
  *out = nullptr;
  whff_status_t st = check_mode(mode, param);
  if (st != WHFF_OK) return st;
  if (rows < 1 || cols < 1)
    return fail(WHFF_ERR_DIMENSION, "codec input must be 2D and nonempty");
  if (lda < cols) return fail(WHFF_ERR_DIMENSION, "lda < cols");
  cudaStream_t cs = (cudaStream_t)stream;
  int dev;
  WCK(cudaGetDevice(&dev));
  const uint64_t br = (rows + 3) / 4, bc = (cols + 3) / 4, nb = br * bc;
  uint64_t *d_lens = nullptr, *d_off = nullptr;
  int* d_ovf = nullptr;
  void* d_tmp = nullptr;
  size_t tmp_bytes = 0;
  whff_dstream* s = nullptr;
  whff_status_t rc = WHFF_OK;
  uint64_t total = 0, last_len = 0, last_off = 0;
  int ovf = 0;
  cudaError_t e = cudaMalloc(&d_lens, nb * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_off, nb * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_ovf, sizeof(int));
  if (e == cudaSuccess) e = cudaMemsetAsync(d_ovf, 0, sizeof(int), cs);
  if (e != cudaSuccess) { rc = cuda_fail(e, "compress alloc"); goto done; }
  k_encode_len<<<grid_for(nb, 128), 128, 0, cs>>>(a, lda, rows, cols, nb, bc, mode, param, d_lens, d_ovf);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_lens, d_off, nb, cs);
  if (e == cudaSuccess) e = cudaMalloc(&d_tmp, tmp_bytes);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_lens, d_off, nb, cs);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&last_len, d_lens + nb - 1, 8, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&last_off, d_off + nb - 1, 8, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&ovf, d_ovf, sizeof(int), cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) { rc = cuda_fail(e, "compress pass 1"); goto done; }
  if (ovf) { rc = fail(WHFF_ERR_OVERFLOW, "internal error: transform coefficient overflow"); goto done; }
  total = last_off + last_len;
  s = new whff_dstream();
  s->device = dev;
  s->mode = mode;
  s->param = param;
  s->rows = rows;
  s->cols = cols;
  s->br = br;
  s->bc = bc;
  s->nb = nb;
  s->gpr = (bc + 31) / 32;
  s->payload_bytes = (total + 7) / 8;
  s->payload_bits = s->payload_bytes * 8;
  s->total_bits = total;
  s->planes_limit = planes_limit_for(mode, param);
  s->has_raw = mode == WHFF_MODE_ACCURACY;
  s->seg_bits = mode == WHFF_MODE_RATE ? (uint32_t)param * 16u : 0u;
  rc = alloc_payload(s, s->payload_bytes);
  if (rc != WHFF_OK) goto done;
  k_encode_emit<<<grid_for(nb, 128), 128, 0, cs>>>(a, lda, rows, cols, nb, bc, mode, param, d_off,
                                                   reinterpret_cast<uint32_t*>(s->d_payload));
  e = cudaGetLastError();
  if (e != cudaSuccess) { rc = cuda_fail(e, "compress pass 2"); goto done; }
  if (mode == WHFF_MODE_RATE) {
    s->kind = WHFF_INDEX_IMPLICIT;
  } else {
    s->kind = WHFF_INDEX_COMPACT;  // encoder segments are <= 1333 bits
    e = cudaMalloc(&s->d_lens, nb * 2);
    if (e == cudaSuccess) e = cudaMalloc(&s->d_base, br * s->gpr * 8);
    if (e != cudaSuccess) { rc = cuda_fail(e, "compress index alloc"); goto done; }
    k_build_compact<<<grid_for(nb, 256), 256, 0, cs>>>(d_off, nb, bc, s->gpr, s->payload_bits,
                                                       s->d_lens, s->d_base);
    s->index_bytes = nb * 2 + br * s->gpr * 8;
  }
  e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) { rc = cuda_fail(e, "compress finish"); goto done; }
done:
  cudaFree(d_lens);
  cudaFree(d_off);
  cudaFree(d_ovf);
  cudaFree(d_tmp);
  if (rc != WHFF_OK) {
    free_stream(s);
    return rc;
  }
  *out = s;
  return WHFF_OK;
}

static EncArrays enc_arrays(const uint32_t* mag, const uint8_t* neg, const uint16_t* emax,
                            const uint8_t* planes, const uint8_t* raw_mask, const uint32_t* raw_words) {
  EncArrays E{mag, neg, emax, planes, raw_mask, raw_words};
  return E;
}

whff_status_t whff_encode_blocks_size(const uint32_t* mag, const uint8_t* neg, const uint16_t* emax,
                                      const uint8_t* planes, const uint8_t* raw_mask,
                                      const uint32_t* raw_words, uint64_t nb, int n_planes,
                                      int budget_bits, int has_raw, uint64_t* offsets,
                                      uint64_t* total_bits, whff_stream_t stream) {
  if (n_planes != kNPlanes) return fail(WHFF_ERR_ARGUMENT, "n_planes must be 27");
  if (!total_bits) return fail(WHFF_ERR_ARGUMENT, "null total_bits");
  *total_bits = 0;
  if (nb == 0) return WHFF_OK;
  cudaStream_t cs = (cudaStream_t)stream;
  uint64_t* d_lens = nullptr;
  void* d_tmp = nullptr;
  size_t tmp_bytes = 0;
  uint64_t last_len = 0, last_off = 0;
  cudaError_t e = cudaMalloc(&d_lens, nb * 8);
  if (e == cudaSuccess) {
    k_encblocks_len<<<grid_for(nb, 128), 128, 0, cs>>>(
        enc_arrays(mag, neg, emax, planes, raw_mask, raw_words), nb, budget_bits, has_raw, d_lens);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_lens, offsets, nb, cs);
  if (e == cudaSuccess) e = cudaMalloc(&d_tmp, tmp_bytes);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_lens, offsets, nb, cs);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&last_len, d_lens + nb - 1, 8, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&last_off, offsets + nb - 1, 8, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  cudaFree(d_lens);
  cudaFree(d_tmp);
  if (e != cudaSuccess) return cuda_fail(e, "encode_blocks pass 1");
  *total_bits = last_off + last_len;
  return WHFF_OK;
}

whff_status_t whff_encode_blocks_emit(const uint32_t* mag, const uint8_t* neg, const uint16_t* emax,
                                      const uint8_t* planes, const uint8_t* raw_mask,
                                      const uint32_t* raw_words, uint64_t nb, int n_planes,
                                      int budget_bits, int has_raw, const uint64_t* offsets,
                                      uint8_t* payload, whff_stream_t stream) {
  if (n_planes != kNPlanes) return fail(WHFF_ERR_ARGUMENT, "n_planes must be 27");
  if (nb == 0) return WHFF_OK;
  if ((reinterpret_cast<uintptr_t>(payload) & 3u) != 0)
    return fail(WHFF_ERR_ARGUMENT, "payload must be 4-byte aligned");
  k_encblocks_emit<<<grid_for(nb, 128), 128, 0, (cudaStream_t)stream>>>(
      enc_arrays(mag, neg, emax, planes, raw_mask, raw_words), nb, budget_bits, has_raw, offsets,
      reinterpret_cast<uint32_t*>(payload));
  WCK_LAUNCH("encode_blocks pass 2");
  return WHFF_OK;
}

whff_status_t whff_decode_blocks(whff_dstream_t s, uint64_t first, uint64_t count, int planes_limit,
                                 uint32_t* mag, uint8_t* neg, uint16_t* emax, uint8_t* raw,
                                 uint32_t* raw_words, uint64_t* consumed, whff_stream_t stream) {
  if (!s) return fail(WHFF_ERR_ARGUMENT, "null stream");
  if (first > s->nb || count > s->nb - first) return fail(WHFF_ERR_CORRUPT, "block index out of range");
  if (count == 0) return WHFF_OK;
  DeviceGuard g(s->device);
  const int pl = planes_limit < 0 ? s->planes_limit : std::min(planes_limit, kNPlanes);
  const StreamView v = s->view();
  cudaStream_t cs = (cudaStream_t)stream;
  if (s->has_raw)
    k_decode_blocks<true><<<grid_for(count, 128), 128, 0, cs>>>(v, first, count, pl, mag, neg, emax,
                                                               raw, raw_words, consumed);
  else
    k_decode_blocks<false><<<grid_for(count, 128), 128, 0, cs>>>(v, first, count, pl, mag, neg, emax,
                                                                raw, raw_words, consumed);
  WCK_LAUNCH("decode_blocks");
  return WHFF_OK;
}

whff_status_t whff_decode_block_words(whff_dstream_t s, uint64_t first, uint64_t count, float* out,
                                      whff_stream_t stream) {
  if (!s || !out) return fail(WHFF_ERR_ARGUMENT, "null argument");
  if (first > s->nb || count > s->nb - first) return fail(WHFF_ERR_CORRUPT, "block index out of range");
  if (count == 0) return WHFF_OK;
  DeviceGuard g(s->device);
  const StreamView v = s->view();
  cudaStream_t cs = (cudaStream_t)stream;
  if (s->has_raw)
    k_decode_block_words<true><<<grid_for(count, 128), 128, 0, cs>>>(v, first, count, out);
  else
    k_decode_block_words<false><<<grid_for(count, 128), 128, 0, cs>>>(v, first, count, out);
  WCK_LAUNCH("decode_block_words");
  return WHFF_OK;
}

whff_status_t whff_decode(whff_dstream_t s, float* out, uint64_t ld, uint64_t* status,
                          whff_stream_t stream) {
  if (!s || !out || !status) return fail(WHFF_ERR_ARGUMENT, "null argument");
  DeviceGuard g(s->device);
  if (ld < s->cols) return fail(WHFF_ERR_DIMENSION, "ld_out < cols");
  const StreamView v = s->view();
  cudaStream_t cs = (cudaStream_t)stream;
  auto* st = reinterpret_cast<unsigned long long*>(status);
  if (s->packed) {
    cudaError_t e = pk_launch_words(pk_view(s), s->pk_nexc, out, ld, st, cs);
    if (e != cudaSuccess) return cuda_fail(e, "decode (packed)");
    return WHFF_OK;
  }
  const uint64_t warps = s->br * s->gpr;
  if (warps == 0) return WHFF_OK;
  const unsigned grid = (unsigned)((warps + 7) / 8);
  const bool sf = s->layout == WHFF_LAYOUT_SKELETON_FIRST;
  if (s->has_raw) {
    if (sf) k_decode_words<true, true><<<grid, 256, 0, cs>>>(v, out, ld, st);
    else k_decode_words<true, false><<<grid, 256, 0, cs>>>(v, out, ld, st);
  } else {
    if (sf) k_decode_words<false, true><<<grid, 256, 0, cs>>>(v, out, ld, st);
    else k_decode_words<false, false><<<grid, 256, 0, cs>>>(v, out, ld, st);
  }
  WCK_LAUNCH("decode");
  return WHFF_OK;
}

}  // extern "C"

// ---- fused decode + GEMV -------------------------------------------------

static int variant_of(const whff_dstream* s) {
  if (s->kind == WHFF_INDEX_IMPLICIT) return s->seg_bits == 128 ? 0 : 1;
  return s->has_raw ? 3 : 2;
}

template <int EVAL, bool SF, int POL>
static void launch_gemv_pol(int var, const JobTable& T, unsigned long long* status,
                            cudaStream_t cs) {
  const unsigned threads = 32 * kGemvWarps;
  const unsigned blocks = (unsigned)(T.total_warps * kSplit);   // kSplit CTAs per block-row
  switch (var) {
    case 0: k_decode_gemv<0, EVAL, SF, POL><<<blocks, threads, 0, cs>>>(T, status); break;
    case 1: k_decode_gemv<1, EVAL, SF, POL><<<blocks, threads, 0, cs>>>(T, status); break;
    case 2: k_decode_gemv<2, EVAL, SF, POL><<<blocks, threads, 0, cs>>>(T, status); break;
    default: k_decode_gemv<3, EVAL, SF, POL><<<blocks, threads, 0, cs>>>(T, status); break;
  }
}

template <int EVAL, bool SF>
static whff_status_t launch_gemv_var(int var, const JobTable& T, int policy,
                                     unsigned long long* status, cudaStream_t cs) {
  if (T.total_warps == 0) return WHFF_OK;
  if (policy == WHFF_POLICY_SINGLE) launch_gemv_pol<EVAL, SF, WHFF_POLICY_SINGLE>(var, T, status, cs);
  else if (EVAL == WHFF_EVAL_COEFF || policy == WHFF_POLICY_MIXED)   // coefficient: mixed/single only
    launch_gemv_pol<EVAL, SF, WHFF_POLICY_MIXED>(var, T, status, cs);
  else launch_gemv_pol<EVAL, SF, (EVAL == WHFF_EVAL_COEFF ? WHFF_POLICY_MIXED : WHFF_POLICY_DOUBLE)>(
      var, T, status, cs);
  WCK_LAUNCH("decode_gemv");
  return WHFF_OK;
}

static whff_status_t launch_gemv(int var, int eval, bool sf, const JobTable& T, int policy,
                                 unsigned long long* status, cudaStream_t cs) {
  if (sf) {
    if (eval == WHFF_EVAL_COEFF) return launch_gemv_var<WHFF_EVAL_COEFF, true>(var, T, policy, status, cs);
    return launch_gemv_var<WHFF_EVAL_EXACT, true>(var, T, policy, status, cs);
  }
  if (eval == WHFF_EVAL_COEFF) return launch_gemv_var<WHFF_EVAL_COEFF, false>(var, T, policy, status, cs);
  return launch_gemv_var<WHFF_EVAL_EXACT, false>(var, T, policy, status, cs);
}

// single-call workspace: [G^T v per block-column (coefficient evaluation)]
// [per-row virtual-warp partials][per-row arrival counters]
static uint64_t align256(uint64_t x) { return (x + 255) & ~255ull; }
static uint64_t ws_u_bytes(const whff_dstream* s, int eval) {
  return (eval == WHFF_EVAL_COEFF || s->packed) ? align256(pad_tiles(s->bc) * sizeof(float4)) : 0;
}
static uint64_t ws_rec_bytes(const whff_dstream* s) {
  return align256(std::max<uint64_t>(s->br, 1) * kVW * sizeof(VwRec));
}

static uint64_t pk_nband(const whff_dstream* s) { return std::max<uint64_t>((s->br + 3) / 4, 1); }
static uint64_t ws_pkrec_bytes(const whff_dstream* s) { return align256(pk_nband(s) * kPkVW * sizeof(PkRec)); }

extern "C" whff_status_t whff_decode_gemv_workspace_size(whff_dstream_t s, int eval, size_t* bytes) {
  if (!s || !bytes) return fail(WHFF_ERR_ARGUMENT, "null argument");
  if (s->packed)
    *bytes = ws_u_bytes(s, eval) + ws_pkrec_bytes(s);
  else
    *bytes = ws_u_bytes(s, eval) + ws_rec_bytes(s) + std::max<uint64_t>(s->br, 1) * sizeof(unsigned);
  return WHFF_OK;
}

static whff_status_t launch_pk(int eval, int policy, const PkTable& T, unsigned long long* status,
                               cudaStream_t cs) {
  cudaError_t e = pk_launch_gemv(eval, policy, T, status, cs);
  if (e != cudaSuccess) return cuda_fail(e, "decode_gemv (packed)");
  return WHFF_OK;
}

static whff_status_t check_policy_eval(int policy, int eval) {
  if (policy < 0 || policy > 2) return fail(WHFF_ERR_ARGUMENT, "unknown precision policy");
  if (eval < 0 || eval > 1) return fail(WHFF_ERR_ARGUMENT, "unknown evaluation");
  if (eval == WHFF_EVAL_COEFF && policy == WHFF_POLICY_DOUBLE)
    return fail(WHFF_ERR_ARGUMENT, "coefficient evaluation supports mixed and single only");
  return WHFF_OK;
}

extern "C" whff_status_t whff_decode_gemv(whff_dstream_t s, const float* v, float* y, int policy, int eval,
                               uint64_t row_begin, uint64_t row_end, void* ws, size_t ws_bytes,
                               uint64_t* status, whff_stream_t stream) {
  if (!s) return fail(WHFF_ERR_ARGUMENT, "null stream");
  whff_status_t st = check_policy_eval(policy, eval);
  if (st != WHFF_OK) return st;
  if (row_begin > row_end || row_end > s->rows) return fail(WHFF_ERR_DIMENSION, "bad row range");
  if (row_begin == row_end) return WHFF_OK;
  if (!v || !y || !status) return fail(WHFF_ERR_ARGUMENT, "null argument");
  DeviceGuard g(s->device);
  cudaStream_t cs = (cudaStream_t)stream;
  if (s->packed) {
    PkTable T;
    T.jobs = nullptr;
    T.prefix = nullptr;
    T.n = 1;
    T.single.p = pk_view(s);
    T.max_nsegb = T.single.p.g.nsegb;
    T.single.v = v;
    T.single.y = y;
    T.single.U = nullptr;
    T.single.row_begin = row_begin;
    T.single.row_end = row_end;
    T.single.band0 = row_begin / 16;
    T.total_bands = (row_end + 15) / 16 - row_begin / 16;
    size_t need = 0;
    whff_decode_gemv_workspace_size(s, eval, &need);
    if (!ws || ws_bytes < need) return fail(WHFF_ERR_ARGUMENT, "workspace too small");
    if ((reinterpret_cast<uintptr_t>(ws) & 15u) != 0) return fail(WHFF_ERR_ARGUMENT, "workspace alignment");
    uint8_t* wsb = reinterpret_cast<uint8_t*>(ws);
    T.recs = reinterpret_cast<PkRec*>(wsb + ws_u_bytes(s, eval));
    vec_prologue(eval, v, s->cols, s->bc, reinterpret_cast<float4*>(ws), cs);
    WCK_LAUNCH("vector prologue");
    T.single.U = reinterpret_cast<const float4*>(ws);
    return launch_pk(eval, policy, T, reinterpret_cast<unsigned long long*>(status), cs);
  }
  JobTable T;
  T.jobs = nullptr;
  T.prefix = nullptr;
  T.row_job = nullptr;
  T.n = 1;
  T.single.s = s->view();
  T.single.v = v;
  T.single.y = y;
  T.single.U = nullptr;
  T.single.row_begin = row_begin;
  T.single.row_end = row_end;
  T.single.br0 = row_begin / 4;
  T.total_warps = (row_end + 3) / 4 - row_begin / 4;
  size_t need = 0;
  whff_decode_gemv_workspace_size(s, eval, &need);
  if (!ws || ws_bytes < need) return fail(WHFF_ERR_ARGUMENT, "workspace too small");
  if ((reinterpret_cast<uintptr_t>(ws) & 15u) != 0) return fail(WHFF_ERR_ARGUMENT, "workspace alignment");
  uint8_t* wsb = reinterpret_cast<uint8_t*>(ws);
  T.recs = reinterpret_cast<VwRec*>(wsb + ws_u_bytes(s, eval));
  T.tickets = reinterpret_cast<unsigned*>(wsb + ws_u_bytes(s, eval) + ws_rec_bytes(s));
  cudaError_t me = cudaMemsetAsync(T.tickets, 0, T.total_warps * sizeof(unsigned), cs);
  if (me != cudaSuccess) return cuda_fail(me, "workspace clear");
  if (eval == WHFF_EVAL_COEFF) {
    k_coeff_prep<<<grid_for(pad_tiles(s->bc), 256), 256, 0, cs>>>(v, s->cols, s->bc, pad_tiles(s->bc),
                                                               reinterpret_cast<float4*>(ws));
    WCK_LAUNCH("coeff_prep");
    T.single.U = reinterpret_cast<const float4*>(ws);
  }
  return launch_gemv(variant_of(s), eval, s->layout == WHFF_LAYOUT_SKELETON_FIRST, T, policy,
                     reinterpret_cast<unsigned long long*>(status), cs);
}

struct whff_gemv_plan {
  int device = 0;
  int n = 0;
  int policy = 0, eval = 0, var = 0;
  bool sf = false;
  GemvJob* d_jobs = nullptr;
  uint64_t* d_prefix = nullptr;
  uint32_t* d_row_job = nullptr;
  uint64_t total_warps = 0;
  float4* d_U = nullptr;
  VwRec* d_recs = nullptr;       // [block-row][kVW] partials
  unsigned* d_tickets = nullptr;  // [block-row] arrival counters (reset by the kernel)
  // packed streams (whff_dstream_pack): band jobs
  bool pk = false;
  uint64_t pk_max_nsegb = 0;      // widest band (segments) of any job
  PkJob* d_pkjobs = nullptr;
  PkRec* d_pkrecs = nullptr;
  // distinct vectors for the coefficient prologue
  std::vector<const float*> prep_v;
  std::vector<uint64_t> prep_cols, prep_bc, prep_off;
  uint64_t bytes_read = 0, bytes_written = 0, n_blocks = 0;
};

// distinct vectors of a plan (coefficient prologue) and their U offsets
static void plan_vectors(whff_gemv_plan* P, int n, const whff_dstream_t* streams, const float* const* v,
                         std::vector<uint64_t>& uoff, uint64_t& ucount) {
  uoff.assign(n, 0);
  ucount = 0;
  for (int i = 0; i < n; ++i) {
    const whff_dstream* s = streams[i];
    int found = -1;
    for (size_t k = 0; k < P->prep_v.size(); ++k)
      if (P->prep_v[k] == v[i] && P->prep_cols[k] == s->cols) found = (int)k;
    if (found < 0) {
      P->prep_v.push_back(v[i]);
      P->prep_cols.push_back(s->cols);
      P->prep_bc.push_back(s->bc);
      P->prep_off.push_back(ucount);
      ucount += pad_tiles(s->bc);
      P->bytes_read += s->cols * 4;
      found = (int)P->prep_v.size() - 1;
    }
    uoff[i] = P->prep_off[found];
  }
}

static whff_status_t plan_create_packed(int n, const whff_dstream_t* streams, const float* const* v,
                                        float* const* y, const uint64_t* rb, const uint64_t* re,
                                        int policy, int eval, whff_gemv_plan_t* out) {
  for (int i = 0; i < n; ++i)
    if (rb[i] > re[i] || re[i] > streams[i]->rows) return fail(WHFF_ERR_DIMENSION, "bad row range");
  whff_gemv_plan* P = new whff_gemv_plan();
  cudaGetDevice(&P->device);
  P->n = n;
  P->policy = policy;
  P->eval = eval;
  P->pk = true;
  std::vector<PkJob> jobs(n);
  std::vector<uint64_t> prefix(n), uoff;
  uint64_t bands = 0, ucount = 0;
  for (int i = 0; i < n; ++i) {
    const whff_dstream* s = streams[i];
    PkJob& J = jobs[i];
    J.p = pk_view(s);
    P->pk_max_nsegb = std::max<uint64_t>(P->pk_max_nsegb, J.p.g.nsegb);
    J.v = v[i];
    J.y = y[i];
    J.U = nullptr;
    J.row_begin = rb[i];
    J.row_end = re[i];
    J.band0 = rb[i] / 16;
    prefix[i] = bands;
    const uint64_t b0 = rb[i] / 16, b1 = rb[i] == re[i] ? b0 : (re[i] + 15) / 16;
    bands += b1 - b0;
    for (uint64_t b = b0; b < b1; ++b) P->bytes_read += s->pk_band_bytes[b];
    P->n_blocks += std::min<uint64_t>(b1 * 4, s->br) * s->bc - std::min<uint64_t>(b0 * 4, s->br) * s->bc;
    P->bytes_written += (re[i] - rb[i]) * 4;
  }
  plan_vectors(P, n, streams, v, uoff, ucount);
  P->total_warps = bands;
  cudaError_t e = cudaSuccess;
  {   // U = G^T v (coefficient) or padded v (exact) per distinct vector
    e = cudaMalloc(&P->d_U, std::max<uint64_t>(ucount, 1) * sizeof(float4));
    for (int i = 0; i < n && e == cudaSuccess; ++i) jobs[i].U = P->d_U + uoff[i];
  }
  if (e == cudaSuccess) e = cudaMalloc(&P->d_pkjobs, n * sizeof(PkJob));
  if (e == cudaSuccess) e = cudaMalloc(&P->d_prefix, n * sizeof(uint64_t));
  if (e == cudaSuccess) e = cudaMemcpy(P->d_pkjobs, jobs.data(), n * sizeof(PkJob), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(P->d_prefix, prefix.data(), n * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&P->d_pkrecs, std::max<uint64_t>(bands, 1) * kPkVW * sizeof(PkRec));
  if (e != cudaSuccess) {
    cudaFree(P->d_U);
    cudaFree(P->d_pkjobs);
    cudaFree(P->d_prefix);
    cudaFree(P->d_pkrecs);
    delete P;
    return cuda_fail(e, "plan create (packed)");
  }
  *out = P;
  return WHFF_OK;
}

extern "C" {

whff_status_t whff_gemv_plan_create(int n, const whff_dstream_t* streams, const float* const* v,
                                    float* const* y, const uint64_t* rb, const uint64_t* re,
                                    int policy, int eval, whff_gemv_plan_t* out) {
  if (!out || n < 1 || !streams || !v || !y || !rb || !re) return fail(WHFF_ERR_ARGUMENT, "bad plan arguments");
  *out = nullptr;
  whff_status_t st = check_policy_eval(policy, eval);
  if (st != WHFF_OK) return st;
  for (int i = 0; i < n; ++i)
    if (!streams[i]) return fail(WHFF_ERR_ARGUMENT, "null stream in plan");
  bool all_packed = true;
  for (int i = 0; i < n; ++i) all_packed = all_packed && streams[i]->packed;
  if (all_packed) return plan_create_packed(n, streams, v, y, rb, re, policy, eval, out);
  const int var = variant_of(streams[0]);
  for (int i = 0; i < n; ++i) {
    if (variant_of(streams[i]) != var || streams[i]->mode != streams[0]->mode ||
        streams[i]->layout != streams[0]->layout)
      return fail(WHFF_ERR_ARGUMENT, "plan streams must share mode, index kind and layout");
    if (rb[i] > re[i] || re[i] > streams[i]->rows) return fail(WHFF_ERR_DIMENSION, "bad row range");
  }
  whff_gemv_plan* P = new whff_gemv_plan();
  cudaGetDevice(&P->device);
  P->n = n;
  P->policy = policy;
  P->eval = eval;
  P->var = var;
  P->sf = streams[0]->layout == WHFF_LAYOUT_SKELETON_FIRST;
  std::vector<GemvJob> jobs(n);
  std::vector<uint64_t> prefix(n), uoff(n, 0);
  uint64_t warps = 0, ucount = 0;
  for (int i = 0; i < n; ++i) {
    const whff_dstream* s = streams[i];
    GemvJob& J = jobs[i];
    J.s = s->view();
    J.v = v[i];
    J.y = y[i];
    J.U = nullptr;
    J.row_begin = rb[i];
    J.row_end = re[i];
    J.br0 = rb[i] / 4;
    prefix[i] = warps;
    const uint64_t nbr = rb[i] == re[i] ? 0 : (re[i] + 3) / 4 - rb[i] / 4;
    warps += nbr;
    // traffic accounting (roofline): payload + index of the covered rows
    const uint64_t blocks = nbr * s->bc;
    P->n_blocks += blocks;
    if (s->kind == WHFF_INDEX_IMPLICIT)
      P->bytes_read += blocks * s->seg_bits / 8;
    else
      P->bytes_read += (uint64_t)((double)s->payload_bytes * blocks / std::max<uint64_t>(s->nb, 1));
    P->bytes_read += (uint64_t)((double)s->index_bytes * blocks / std::max<uint64_t>(s->nb, 1));
    P->bytes_written += (re[i] - rb[i]) * 4;
    // distinct vectors
    int found = -1;
    for (size_t k = 0; k < P->prep_v.size(); ++k)
      if (P->prep_v[k] == v[i] && P->prep_cols[k] == s->cols) found = (int)k;
    if (found < 0) {
      P->prep_v.push_back(v[i]);
      P->prep_cols.push_back(s->cols);
      P->prep_bc.push_back(s->bc);
      P->prep_off.push_back(ucount);
      ucount += pad_tiles(s->bc);
      P->bytes_read += s->cols * 4;
      found = (int)P->prep_v.size() - 1;
    }
    uoff[i] = P->prep_off[found];
  }
  P->total_warps = warps;
  cudaError_t e = cudaSuccess;
  if (eval == WHFF_EVAL_COEFF) {
    e = cudaMalloc(&P->d_U, std::max<uint64_t>(ucount, 1) * sizeof(float4));
    for (int i = 0; i < n && e == cudaSuccess; ++i) jobs[i].U = P->d_U + uoff[i];
  }
  if (e == cudaSuccess) e = cudaMalloc(&P->d_jobs, n * sizeof(GemvJob));
  if (e == cudaSuccess) e = cudaMalloc(&P->d_prefix, n * sizeof(uint64_t));
  if (e == cudaSuccess) e = cudaMemcpy(P->d_jobs, jobs.data(), n * sizeof(GemvJob), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(P->d_prefix, prefix.data(), n * 8, cudaMemcpyHostToDevice);
  {
    std::vector<uint32_t> row_job(std::max<uint64_t>(warps, 1), 0u);
    for (int i = 0; i < n; ++i) {
      const uint64_t end = i + 1 < n ? prefix[i + 1] : warps;
      for (uint64_t r = prefix[i]; r < end; ++r) row_job[r] = (uint32_t)i;
    }
    if (e == cudaSuccess) e = cudaMalloc(&P->d_row_job, row_job.size() * sizeof(uint32_t));
    if (e == cudaSuccess)
      e = cudaMemcpy(P->d_row_job, row_job.data(), row_job.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) e = cudaMalloc(&P->d_recs, std::max<uint64_t>(warps, 1) * kVW * sizeof(VwRec));
  if (e == cudaSuccess) e = cudaMalloc(&P->d_tickets, std::max<uint64_t>(warps, 1) * sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemset(P->d_tickets, 0, std::max<uint64_t>(warps, 1) * sizeof(unsigned));
  if (e != cudaSuccess) {
    cudaFree(P->d_U);
    cudaFree(P->d_jobs);
    cudaFree(P->d_prefix);
    cudaFree(P->d_row_job);
    cudaFree(P->d_recs);
    cudaFree(P->d_tickets);
    delete P;
    return cuda_fail(e, "plan create");
  }
  *out = P;
  return WHFF_OK;
}

whff_status_t whff_gemv_plan_launch(whff_gemv_plan_t P, uint64_t* status, whff_stream_t stream) {
  if (!P || !status) return fail(WHFF_ERR_ARGUMENT, "null argument");
  DeviceGuard g(P->device);
  cudaStream_t cs = (cudaStream_t)stream;
  if (P->eval == WHFF_EVAL_COEFF || P->pk) {
    for (size_t k = 0; k < P->prep_v.size(); ++k)
      vec_prologue(P->eval, P->prep_v[k], P->prep_cols[k], P->prep_bc[k], P->d_U + P->prep_off[k], cs);
    WCK_LAUNCH("plan vector prologue");
  }
  if (P->pk) {
    PkTable T;
    T.jobs = P->d_pkjobs;
    T.prefix = P->d_prefix;
    T.n = P->n;
    T.total_bands = P->total_warps;
    T.max_nsegb = P->pk_max_nsegb;
    memset(&T.single, 0, sizeof(T.single));
    T.recs = P->d_pkrecs;
    return launch_pk(P->eval, P->policy, T, reinterpret_cast<unsigned long long*>(status), cs);
  }
  JobTable T;
  T.jobs = P->d_jobs;
  T.prefix = P->d_prefix;
  T.row_job = P->d_row_job;
  T.n = P->n;
  T.total_warps = P->total_warps;
  memset(&T.single, 0, sizeof(T.single));
  T.recs = P->d_recs;
  T.tickets = P->d_tickets;
  return launch_gemv(P->var, P->eval, P->sf, T, P->policy, reinterpret_cast<unsigned long long*>(status), cs);
}

whff_status_t whff_gemv_plan_traffic(whff_gemv_plan_t P, uint64_t* br, uint64_t* bw, uint64_t* nb) {
  if (!P) return fail(WHFF_ERR_ARGUMENT, "null plan");
  if (br) *br = P->bytes_read;
  if (bw) *bw = P->bytes_written;
  if (nb) *nb = P->n_blocks;
  return WHFF_OK;
}

whff_status_t whff_gemv_plan_destroy(whff_gemv_plan_t P) {
  if (!P) return WHFF_OK;
  DeviceGuard g(P->device);
  cudaFree(P->d_U);
  cudaFree(P->d_jobs);
  cudaFree(P->d_prefix);
  cudaFree(P->d_row_job);
  cudaFree(P->d_recs);
  cudaFree(P->d_tickets);
  cudaFree(P->d_pkjobs);
  cudaFree(P->d_pkrecs);
  delete P;
  return WHFF_OK;
}

}  // extern "C"

// ---- dense GEMV -----------------------------------------------------------

static void blocked_split(uint64_t rows, uint64_t cols, uint64_t& nseg, uint64_t& seg_cols) {
  // enough warps for 148 SMs x 64 warps; segments a multiple of one batch of
  // kBlkU float4 per lane (512 columns)
  constexpr uint64_t kSeg = 128 * kBlkU;
  const uint64_t target = 148ull * 64;
  nseg = rows >= target ? 1 : (target + rows - 1) / rows;
  const uint64_t max_seg = std::max<uint64_t>(1, (cols + kSeg - 1) / kSeg);
  nseg = std::min(nseg, max_seg);
  seg_cols = ((cols + nseg - 1) / nseg + kSeg - 1) / kSeg * kSeg;
  nseg = (cols + seg_cols - 1) / seg_cols;
  if (nseg == 0) nseg = 1;
}

extern "C" whff_status_t whff_gemv_workspace_size(uint64_t rows, uint64_t cols, int policy, int shape, int fanout,
                                       size_t* bytes) {
  if (!bytes) return fail(WHFF_ERR_ARGUMENT, "null argument");
  *bytes = 0;
  if (shape == WHFF_SHAPE_FIXED_TREE) {
    if (fanout < 2 || (fanout & (fanout - 1))) return fail(WHFF_ERR_ARGUMENT, "tree fanout must be a power of two >= 2");
    const uint64_t ng = (cols + fanout - 1) / fanout;
    const size_t el = policy == WHFF_POLICY_SINGLE ? 4 : 8;
    *bytes = 2 * rows * std::max<uint64_t>(ng, 1) * el + 256;
  } else if (shape == WHFF_SHAPE_BLOCKED) {
    uint64_t nseg, segc;
    blocked_split(rows, cols, nseg, segc);
    *bytes = rows * nseg * 8;
  }
  return WHFF_OK;
}

template <int POL>
static whff_status_t gemv_pol(const float* A, uint64_t lda, uint64_t rows, uint64_t cols,
                              const float* v, float* y, int shape, int fanout, void* ws, size_t wsb,
                              cudaStream_t cs) {
  if (shape == WHFF_SHAPE_SEQUENTIAL) {
    if (seq_staged_ok(A, lda, v)) {
      static std::atomic<uint64_t> attr{0};
      WCK(ensure_dyn_smem(k_gemv_seq_staged<POL>, kSqWarps * sq_warp_bytes(32), attr));
      const int nr = seq_rows_per_warp(rows);
      const uint64_t nw = (rows + nr - 1) / nr;
      k_gemv_seq_staged<POL><<<(unsigned)((nw + kSqWarps - 1) / kSqWarps), 32 * kSqWarps, kSqWarps * sq_warp_bytes(nr),
                               cs>>>(A, lda, rows, cols, v, y, nr);
    } else {
      k_gemv_seq<POL, false><<<grid_for(rows, 64), 64, 0, cs>>>(A, lda, rows, cols, v, y, nullptr);
    }
    WCK_LAUNCH("gemv sequential");
    return WHFF_OK;
  }
  size_t need = 0;
  whff_status_t st = whff_gemv_workspace_size(rows, cols, POL, shape, fanout, &need);
  if (st != WHFF_OK) return st;
  if (wsb < need || (need && !ws)) return fail(WHFF_ERR_ARGUMENT, "workspace too small");
  if (shape == WHFF_SHAPE_FIXED_TREE) {
    using T = typename std::conditional<POL == WHFF_POLICY_SINGLE, float, double>::type;
    T* b0 = reinterpret_cast<T*>(ws);
    uint64_t ng = (cols + fanout - 1) / fanout;
    T* b1 = b0 + rows * std::max<uint64_t>(ng, 1);
    k_gemv_tree_leaf<POL, T><<<grid_for(rows * ng, 256), 256, 0, cs>>>(A, lda, rows, cols, v, fanout, b0, ng);
    WCK_LAUNCH("gemv tree leaf");
    uint64_t w = ng;
    while (w > 1) {
      const uint64_t n2 = (w + fanout - 1) / fanout;
      k_gemv_tree_level<T><<<grid_for(rows * n2, 256), 256, 0, cs>>>(b0, rows, w, fanout, b1, n2);
      WCK_LAUNCH("gemv tree level");
      std::swap(b0, b1);
      w = n2;
    }
    k_tree_store<T><<<grid_for(rows, 256), 256, 0, cs>>>(b0, rows, y);
    WCK_LAUNCH("gemv tree store");
    return WHFF_OK;
  }
  if (shape != WHFF_SHAPE_BLOCKED) return fail(WHFF_ERR_ARGUMENT, "unknown reduction shape");
  uint64_t nseg, segc;
  blocked_split(rows, cols, nseg, segc);
  const bool vec4 = (lda % 4 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15u) == 0) &&
                    ((reinterpret_cast<uintptr_t>(v) & 15u) == 0);
  k_gemv_blocked<POL><<<grid_for(rows * nseg * 32, 256), 256, 0, cs>>>(
      A, lda, rows, cols, v, nseg, segc, vec4, reinterpret_cast<double*>(ws));
  WCK_LAUNCH("gemv blocked");
  k_blocked_finish<POL><<<grid_for(rows, 256), 256, 0, cs>>>(reinterpret_cast<double*>(ws), rows, nseg, y);
  WCK_LAUNCH("gemv blocked finish");
  return WHFF_OK;
}

extern "C" {

whff_status_t whff_gemv(const float* A, uint64_t lda, uint64_t rows, uint64_t cols, const float* v,
                        float* y, int policy, int shape, int fanout, void* ws, size_t wsb,
                        whff_stream_t stream) {
  if (!A || !v || !y) return fail(WHFF_ERR_ARGUMENT, "null argument");
  if (rows < 1 || cols < 1) return fail(WHFF_ERR_DIMENSION, "gemv operands must be nonempty");
  if (lda < cols) return fail(WHFF_ERR_DIMENSION, "lda < cols");
  cudaStream_t cs = (cudaStream_t)stream;
  switch (policy) {
    case WHFF_POLICY_MIXED: return gemv_pol<WHFF_POLICY_MIXED>(A, lda, rows, cols, v, y, shape, fanout, ws, wsb, cs);
    case WHFF_POLICY_SINGLE: return gemv_pol<WHFF_POLICY_SINGLE>(A, lda, rows, cols, v, y, shape, fanout, ws, wsb, cs);
    case WHFF_POLICY_DOUBLE: return gemv_pol<WHFF_POLICY_DOUBLE>(A, lda, rows, cols, v, y, shape, fanout, ws, wsb, cs);
  }
  return fail(WHFF_ERR_ARGUMENT, "unknown precision policy");
}

whff_status_t whff_gemv_oracle(const float* A, uint64_t lda, uint64_t rows, uint64_t cols,
                               const float* v, double* y, whff_stream_t stream) {
  if (!A || !v || !y) return fail(WHFF_ERR_ARGUMENT, "null argument");
  if (rows < 1 || cols < 1) return fail(WHFF_ERR_DIMENSION, "gemv operands must be nonempty");
  k_gemv_seq<WHFF_POLICY_DOUBLE, true><<<grid_for(rows, 64), 64, 0, (cudaStream_t)stream>>>(
      A, lda, rows, cols, v, nullptr, y);
  WCK_LAUNCH("gemv oracle");
  return WHFF_OK;
}

whff_status_t whff_gemv_oracle_f64(const double* A, uint64_t lda, uint64_t rows, uint64_t cols,
                                   const double* v, double* y, whff_stream_t stream) {
  if (!A || !v || !y) return fail(WHFF_ERR_ARGUMENT, "null argument");
  if (rows < 1 || cols < 1) return fail(WHFF_ERR_DIMENSION, "gemv operands must be nonempty");
  k_gemv_oracle64<<<grid_for(rows, 64), 64, 0, (cudaStream_t)stream>>>(A, lda, rows, cols, v, y);
  WCK_LAUNCH("gemv oracle f64");
  return WHFF_OK;
}

whff_status_t whff_find_nonfinite(const float* x, uint64_t n, uint64_t* status, whff_stream_t stream) {
  if (!status) return fail(WHFF_ERR_ARGUMENT, "null status");
  if (n == 0) return WHFF_OK;
  const unsigned blocks = (unsigned)std::min<uint64_t>(grid_for(n, 256), 148ull * 8);
  k_find_nonfinite<<<blocks, 256, 0, (cudaStream_t)stream>>>(x, n, reinterpret_cast<unsigned long long*>(status));
  WCK_LAUNCH("find_nonfinite");
  return WHFF_OK;
}

whff_status_t whff_csr_matvec(const int64_t* indptr, const int32_t* indices, const double* data,
                              uint64_t n, const float* x, const float* b, const float* u, float* y,
                              whff_stream_t stream) {
  if (!indptr || !x || !y) return fail(WHFF_ERR_ARGUMENT, "null argument");
  if ((b == nullptr) != (u == nullptr)) return fail(WHFF_ERR_ARGUMENT, "b and u go together");
  if (n == 0) return WHFF_OK;
  k_csr_matvec<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(indptr, indices, data, n, x, b, u, y);
  WCK_LAUNCH("csr_matvec");
  return WHFF_OK;
}

whff_status_t whff_device_timestamp(uint64_t* t_dev, whff_stream_t stream) {
  if (!t_dev) return fail(WHFF_ERR_ARGUMENT, "null argument");
  k_timestamp<<<1, 1, 0, (cudaStream_t)stream>>>(t_dev);
  WCK_LAUNCH("device_timestamp");
  return WHFF_OK;
}

whff_status_t whff_wait_until(const uint64_t* base_dev, uint64_t offset_ns, whff_stream_t stream) {
  if (!base_dev) return fail(WHFF_ERR_ARGUMENT, "null argument");
  k_wait_until<<<1, 1, 0, (cudaStream_t)stream>>>(base_dev, offset_ns);
  WCK_LAUNCH("wait_until");
  return WHFF_OK;
}

whff_status_t whff_source_term(const float* fp, const float* dark, float dose, uint64_t n, float* u,
                               whff_stream_t stream) {
  if (!dark || !u) return fail(WHFF_ERR_ARGUMENT, "null argument");
  if (n == 0) return WHFF_OK;
  k_source_term<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(fp, dark, dose, n, u);
  WCK_LAUNCH("source_term");
  return WHFF_OK;
}

}  // extern "C"
