// whff_packed_api.h -- what whff_b200.cu (streams, plans, the C ABI) needs
// from the packed-layout translation unit (whff_packed.cu): the device-side
// views / job tables and the host launchers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "whff_packed.cuh"

// ---------------------------------------------------------------------------
// device view of a packed stream
// ---------------------------------------------------------------------------
struct PkView {
  const uint32_t* body;
  const whff::pk::Seg* segs;          // [band][segment]
  const whff::pk::FieldPar* pars;     // [band][segment][16]: seg_param (k_pk_gemv2)
  const uint64_t* exc_block;    // [exception] block index (row-major blocks)
  const uint32_t* exc_words;    // [exception][16] binary32 words, raster order
  whff::pk::Geom g;
};

struct PkJob {
  PkView p;
  const float* v;
  const float4* U;     // coefficient domain: G^T v per block-column
  float* y;
  uint64_t row_begin, row_end;
  uint64_t band0;      // first band of the job
};

// per-(band, virtual warp) partial sums: 16 rows of a band
struct PkRec {
  double d[16];   // mixed/double: coefficient-domain (or spatial) sums
  double r[16];   //   exception (spatial) sums
  float f[16];    // single
  float rf[16];
};

struct PkTable {
  const PkJob* jobs;         // device table (plans) or nullptr
  const uint64_t* prefix;    // first band of each job
  int n;
  uint64_t total_bands;
  uint64_t max_nsegb;        // widest band of any job, in segments (kernel choice)
  PkJob single;
  PkRec* recs;               // [band][kVW] partial records (k_pk_gemv2 -> k_pk_combine)
};


constexpr int kPkVW = 32;                   // virtual warps per band

// host launchers (whff_packed.cu); all asynchronous on `cs`
cudaError_t pk_launch_stats(const struct StreamView& s, const whff::pk::Geom& g, whff::pk::Seg* segs,
                            uint64_t* seg_words, uint64_t* seg_exc, cudaStream_t cs);
// segment headers followed by the per-segment parameter tables
inline uint64_t pk_segs_bytes(uint64_t nseg) {
  return nseg * (sizeof(whff::pk::Seg) + 16 * sizeof(whff::pk::FieldPar));
}
cudaError_t pk_launch_params(whff::pk::Seg* segs, uint64_t nseg, cudaStream_t cs);
cudaError_t pk_launch_finalize(whff::pk::Seg* segs, uint64_t nseg, const uint64_t* off, const uint64_t* eoff,
                               cudaStream_t cs);
cudaError_t pk_launch_emit(const struct StreamView& s, const whff::pk::Geom& g, const whff::pk::Seg* segs,
                           uint32_t* body, uint64_t* exc_block, uint32_t* exc_words, cudaStream_t cs);
cudaError_t pk_launch_words(const PkView& v, uint64_t nexc, float* out, uint64_t ld,
                            unsigned long long* status, cudaStream_t cs);
cudaError_t pk_launch_gemv(int eval, int policy, const PkTable& T, unsigned long long* status,
                           cudaStream_t cs);
