/*
 * whff_b200.h -- C ABI of the B200-native WHFF hot path (libwhff_b200.so).
 *
 * Drop-in boundary for the reference's kernel plugin contract
 * (whff/backend.py:36-46: a module exposing NAME, gemv_kernel,
 * encode_blocks, decode_blocks) and for the device-resident parts of the
 * codec / GEMV API the reference implements in Python on top of it.
 * Each entry point cites the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/whff/; K = _kernels.pyx).
 *
 * Conventions
 *  - Plain pointers and sizes only.  "dev" pointers are CUDA device memory of
 *    the calling thread's current device; "host" pointers are host memory.
 *  - Every compute call is asynchronous on the caller's stream
 *    (whff_stream_t == cudaStream_t, NULL = legacy default stream) unless
 *    documented as synchronous, and returns a whff_status_t.
 *  - Device-detected data errors (non-finite decoded values) are reported
 *    through a caller-owned device word `status_dev` (uint64, initialise to
 *    WHFF_STATUS_CLEAR); after the stream is synchronised a value other than
 *    WHFF_STATUS_CLEAR is the smallest flat index of a non-finite value.
 *  - Outputs and workspaces are caller-owned; no allocation happens on the
 *    hot path (decode / decode_gemv / gemv / plan launch).  Stream objects and
 *    plans own their device memory (allocated at create, freed at destroy).
 *  - Thread-safe across distinct handles and streams (no global mutable
 *    state apart from the thread-local last-error message).
 *  - Status codes map 1:1 onto errors.py:
 *      WHFF_ERR_DIMENSION -> DimensionError      WHFF_ERR_NONFINITE -> NonFiniteError
 *      WHFF_ERR_CORRUPT   -> CorruptStreamError  WHFF_ERR_ARGUMENT  -> WhffError
 *      WHFF_ERR_OVERFLOW  -> WhffError (codec.py:240-241)
 *      WHFF_ERR_NOMEM     -> MemoryError (K:105,118,254)
 *      WHFF_ERR_CUDA      -> RuntimeError (device failure)
 */
#ifndef WHFF_B200_H
#define WHFF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WHFF_ABI_VERSION 2
#define WHFF_STATUS_CLEAR UINT64_MAX

typedef struct CUstream_st* whff_stream_t; /* == cudaStream_t */
typedef struct whff_dstream* whff_dstream_t;
typedef struct whff_gemv_plan* whff_gemv_plan_t;

typedef enum whff_status {
  WHFF_OK = 0,
  WHFF_ERR_DIMENSION = 1,
  WHFF_ERR_NONFINITE = 2,
  WHFF_ERR_CORRUPT = 3,
  WHFF_ERR_ARGUMENT = 4,
  WHFF_ERR_OVERFLOW = 5,
  WHFF_ERR_NOMEM = 6,
  WHFF_ERR_CUDA = 7
} whff_status_t;

/* codec.py:35-37 */
typedef enum whff_mode { WHFF_MODE_RATE = 0, WHFF_MODE_PRECISION = 1, WHFF_MODE_ACCURACY = 2 } whff_mode_t;
/* mpgemv.py:20 POLICIES */
typedef enum whff_policy { WHFF_POLICY_MIXED = 0, WHFF_POLICY_SINGLE = 1, WHFF_POLICY_DOUBLE = 2 } whff_policy_t;
/* mpgemv.py:21 SHAPES, plus the B200-native deterministic blocked order */
typedef enum whff_shape {
  WHFF_SHAPE_SEQUENTIAL = 0, /* strict left-to-right, bit-exact with K:24-47   */
  WHFF_SHAPE_FIXED_TREE = 1, /* fixed-fanout tree, bit-exact with K:50-77       */
  WHFF_SHAPE_BLOCKED = 2     /* B200 fast path: fixed split + butterfly order   */
} whff_shape_t;
/* how the fused decode+GEMV evaluates a block */
typedef enum whff_eval {
  WHFF_EVAL_EXACT = 0, /* bit-exact decoded words x, binary32 products x*v    */
  WHFF_EVAL_COEFF = 1  /* coefficient domain: y = G * sum 2^(e-26) Q (G^T v)  */
} whff_eval_t;
/* device payload layout (whff_dstream_relayout) */
typedef enum whff_layout {
  WHFF_LAYOUT_REFERENCE = 0,      /* WHFZ bytes as produced by codec.compress        */
  WHFF_LAYOUT_SKELETON_FIRST = 1  /* per-block bit permutation: header, significance
                                     skeleton, then refinement bits per coefficient;
                                     same bytes/index, decodes to identical words    */
} whff_layout_t;
/* device index layout chosen at stream creation */
typedef enum whff_index_kind {
  WHFF_INDEX_IMPLICIT = 0, /* fixed rate, offsets b*16*bpv: no index bytes   */
  WHFF_INDEX_COMPACT = 1,  /* u64 base per 32 blocks of a block-row + u16 len */
  WHFF_INDEX_FULL = 2      /* u64 start + u16 len per block                   */
} whff_index_kind_t;

typedef struct whff_dstream_info {
  int32_t mode;
  int32_t index_kind;
  double param;
  uint64_t rows, cols, n_blocks;
  uint64_t payload_bytes;  /* as uploaded (reference payload.size)            */
  uint64_t total_bits;     /* exact for GPU-encoded streams, else payload bits*/
  uint64_t index_bytes;    /* device index bytes read by a full decode        */
  uint64_t device_bytes;   /* all device memory owned by the stream           */
  int32_t planes_limit;
  int32_t has_raw_flag;
  int32_t layout;          /* whff_layout_t */
  int32_t packed;          /* 1: the tile-packed copy exists (whff_dstream_pack) */
  uint64_t packed_bytes;   /* bytes of the packed copy a full GEMV reads      */
  uint64_t packed_exceptions; /* blocks held as exact words in its side list   */
  int32_t device;          /* CUDA device the stream's memory lives on          */
} whff_dstream_info_t;

int whff_abi_version(void);
const char* whff_status_string(whff_status_t s);
/* thread-local detail message of the last failing call on this thread */
const char* whff_last_error(void);

/* ------------------------------------------------------------------ */
/* Device-resident compressed streams                                  */
/* ------------------------------------------------------------------ */

/* Upload a reference stream (codec.py:71-91 CompressedStream, or the WHFZ
 * file read by codec.py:412-450 load_stream) to `device`.  Validates like
 * codec.py:347-356 (_validate_stream) and :335-344 (_segment_lengths) and
 * builds the device index.  Synchronous.                                   */
whff_status_t whff_dstream_create(int device, int mode, double param,
                                  uint64_t rows, uint64_t cols,
                                  const uint8_t* payload_host, uint64_t payload_bytes,
                                  const uint64_t* block_index_host, uint64_t n_blocks,
                                  whff_dstream_t* out);
/* Segment-table stream for the plugin-level decode_blocks (K:371-408),
 * whose caller supplies explicit offsets/seglens (codec.py:304-306, :327-330)
 * rather than a full stream.  Shape is 4 x 4*n_blocks.  Synchronous.      */
whff_status_t whff_dstream_create_segments(int device, const uint8_t* payload_host,
                                           uint64_t payload_bytes, const uint64_t* offsets_host,
                                           const uint64_t* seglens_host, uint64_t n_blocks,
                                           int planes_limit, int has_raw_flag,
                                           whff_dstream_t* out);
whff_status_t whff_dstream_destroy(whff_dstream_t s);
/* Re-lay the device payload out in place (forward or inverse permutation of
 * every block segment, computed by the reference parse on the device).
 * Needs an implicit or compact index (disjoint segments).  Synchronous.    */
whff_status_t whff_dstream_relayout(whff_dstream_t s, int layout, whff_stream_t stream);
/* Build the stream's tile-packed device copy (csrc/whff_packed.cuh): the
 * decoded coefficients of every block -- exactly the fields decode_blocks
 * (K:371-408) yields -- re-coded losslessly as fixed-width fields per
 * 4-block-row x 256-block-column segment, plus an exact-word side list for
 * raw-escape / extreme-scale blocks.  Decoded words stay bit-exact; every
 * decode / decode_gemv / plan call on a packed stream reads the packed copy
 * (the WHFZ payload stays for download, decode_blocks and relayout).  A
 * rebind / import drops it.  Synchronous on `stream`.                     */
whff_status_t whff_dstream_pack(whff_dstream_t s, whff_stream_t stream);
/* The packed copy to host memory (tooling / tests): segment headers (48 B
 * each), body words, exception block indices and words (16 u32 each).
 * NULL buffers: only the counts are returned.  Synchronous.               */
whff_status_t whff_dstream_packed_download(whff_dstream_t s, uint8_t* segs_host, uint32_t* body_host,
                                           uint64_t* exc_block_host, uint32_t* exc_words_host,
                                           uint64_t* n_segs, uint64_t* body_words, uint64_t* n_exc);
/* Physically distinct device copy of a stream (same device).  Synchronous. */
whff_status_t whff_dstream_clone(whff_dstream_t s, whff_dstream_t* out);
whff_status_t whff_dstream_get_info(whff_dstream_t s, whff_dstream_info_t* info);
/* Start bit of every block-row in the WHFZ payload, out_host[0..br] (br =
 * ceil(rows/4); out_host[br] = payload bits).  Block-rows are contiguous in
 * the stream (codec.py:157-164), so out[b+1] - out[b] is the compressed size
 * of block-row b: the weight of the byte-balanced row sharding
 * (executor.shard_units).  Synchronous.                         */
whff_status_t whff_dstream_block_row_bits(whff_dstream_t s, uint64_t* out_host);
/* Copy payload (payload_bytes) and u64 block bit offsets (n_blocks) back to
 * the host, e.g. for codec.py:388-402 save_stream.  Synchronous.           */
/* Streaming scan staging (pipeline.py:208-289 stage 1, the paper's transfer
 * stage).  export: the stream's device-layout payload and index arrays
 * (compact: base u64[br*gpr] + lens u16[nb]; full: starts u64[nb] + lens
 * u16[nb]; implicit: none) to host memory -- pass NULL buffers to query the
 * sizes.  reserve: grow a stream's payload capacity.  import_async: rebind a
 * slot stream (same rows, cols, mode, index kind; payload within capacity)
 * to exported contents: its geometry (payload size) changes immediately --
 * plans created afterwards see it -- and the bytes are copied in `stream`
 * order (pinned host memory for an asynchronous copy).                     */
whff_status_t whff_dstream_export(whff_dstream_t s, uint8_t* payload_host, uint64_t* payload_bytes,
                                  uint8_t* index_host, uint64_t* index_bytes);
whff_status_t whff_dstream_reserve(whff_dstream_t s, uint64_t payload_capacity);
/* the geometry part of import_async alone (no copy)                        */
whff_status_t whff_dstream_rebind(whff_dstream_t s, uint64_t payload_bytes);
whff_status_t whff_dstream_import_async(whff_dstream_t s, const uint8_t* payload_host,
                                        uint64_t payload_bytes, const uint8_t* index_host,
                                        uint64_t index_bytes, whff_stream_t stream);
whff_status_t whff_dstream_download(whff_dstream_t s, uint8_t* payload_host,
                                    uint64_t* block_index_host);

/* ------------------------------------------------------------------ */
/* Codec: encode (codec.py:225-268 compress; K:228-283 encode_blocks)   */
/* ------------------------------------------------------------------ */

/* GPU compress of a row-major float32 device matrix (pitch lda elements)
 * into a new device stream.  Synchronous on `stream`.  Input must be finite
 * (codec.py:231-232 is checked by the caller via whff_find_nonfinite).     */
whff_status_t whff_compress(const float* a_dev, uint64_t lda, uint64_t rows, uint64_t cols,
                            int mode, double param, whff_stream_t stream,
                            whff_dstream_t* out);

/* Plugin-level encode_blocks (K:228-283) from per-block coefficient arrays.
 * Pass 1: per-block bit offsets (offsets_dev, nb) and the total bit count. */
whff_status_t whff_encode_blocks_size(const uint32_t* mag_dev, const uint8_t* neg_dev,
                                      const uint16_t* emax_dev, const uint8_t* planes_dev,
                                      const uint8_t* raw_mask_dev, const uint32_t* raw_words_dev,
                                      uint64_t n_blocks, int n_planes, int budget_bits,
                                      int has_raw_flag, uint64_t* offsets_dev,
                                      uint64_t* total_bits_host, whff_stream_t stream);
/* Pass 2: emit into a zeroed device payload of >= ceil(total/8)+16 bytes.  */
whff_status_t whff_encode_blocks_emit(const uint32_t* mag_dev, const uint8_t* neg_dev,
                                      const uint16_t* emax_dev, const uint8_t* planes_dev,
                                      const uint8_t* raw_mask_dev, const uint32_t* raw_words_dev,
                                      uint64_t n_blocks, int n_planes, int budget_bits,
                                      int has_raw_flag, const uint64_t* offsets_dev,
                                      uint8_t* payload_dev, whff_stream_t stream);

/* ------------------------------------------------------------------ */
/* Codec: decode                                                        */
/* ------------------------------------------------------------------ */

/* Parity hook with exactly K:371-408 decode_blocks' outputs for blocks
 * [first_block, first_block+count): mag u32[count*16], neg u8[count*16],
 * emax u16[count], raw u8[count], raw_words u32[count*16],
 * consumed u64[count] (all device).  planes_limit < 0: the stream's own
 * (codec.py:301-303); n_planes is fixed at 27 (codec.py:28).              */
whff_status_t whff_decode_blocks(whff_dstream_t s, uint64_t first_block, uint64_t count,
                                 int planes_limit, uint32_t* mag_dev, uint8_t* neg_dev,
                                 uint16_t* emax_dev, uint8_t* raw_dev, uint32_t* raw_words_dev,
                                 uint64_t* consumed_dev, whff_stream_t stream);

/* Reconstructed 4x4 blocks (codec.py:209-218 _reconstruct_blocks) for
 * blocks [first_block, first_block+count): out_dev float32[count*16] raster
 * order -- the device half of codec.py:317-332 decode_block.             */
whff_status_t whff_decode_block_words(whff_dstream_t s, uint64_t first_block, uint64_t count,
                                      float* out_dev, whff_stream_t stream);

/* codec.py:296-314 decompress: float32 words, bit-exact, into out_dev
 * (rows x cols, row pitch ld_out elements).  Non-finite decoded values are
 * reported through status_dev (codec.py:312-313 -> CorruptStreamError).    */
whff_status_t whff_decode(whff_dstream_t s, float* out_dev, uint64_t ld_out,
                          uint64_t* status_dev, whff_stream_t stream);

/* ------------------------------------------------------------------ */
/* Fused decompress + GEMV (replaces codec.decompress followed by        */
/* mpgemv.gemv, pipeline.py:146 + :199-205)                             */
/* ------------------------------------------------------------------ */

/* y[r - row_begin] = sum_j C[r, j] * v[j] for r in [row_begin, row_end),
 * C the decoded stream.  v_dev has `cols` floats, y_dev row_end-row_begin.
 * workspace: whff_decode_gemv_workspace_size bytes of device memory, 16-byte
 * aligned, any contents (the per-band partial sums; the stream layouts also
 * keep arrival counters there; the coefficient evaluation also G^T v).  A row's result does not depend on
 * the row range or on batching (plans give the same bits).  Calls sharing a
 * workspace must be ordered (one stream).                                  */
whff_status_t whff_decode_gemv_workspace_size(whff_dstream_t s, int eval, size_t* bytes);
whff_status_t whff_decode_gemv(whff_dstream_t s, const float* v_dev, float* y_dev,
                               int policy, int eval, uint64_t row_begin, uint64_t row_end,
                               void* workspace_dev, size_t workspace_bytes,
                               uint64_t* status_dev, whff_stream_t stream);

/* Batched plan: n jobs (stream, vector, output, row range) executed by one
 * launch per call -- the per-light-step deformation products of
 * pipeline.py:199-205 over many slit streams.  Creation builds the device
 * job table and the plan's workspace (synchronous); launch is capture-safe
 * (CUDA graphs); launches of one plan must be ordered (one stream).  All
 * streams of a plan must share mode, index kind and raw flag.             */
whff_status_t whff_gemv_plan_create(int n_jobs, const whff_dstream_t* streams,
                                    const float* const* v_dev, float* const* y_dev,
                                    const uint64_t* row_begin, const uint64_t* row_end,
                                    int policy, int eval, whff_gemv_plan_t* out);
whff_status_t whff_gemv_plan_launch(whff_gemv_plan_t plan, uint64_t* status_dev,
                                    whff_stream_t stream);
/* bytes the plan's launch reads (payload + index + vectors) and writes    */
whff_status_t whff_gemv_plan_traffic(whff_gemv_plan_t plan, uint64_t* bytes_read,
                                     uint64_t* bytes_written, uint64_t* n_blocks);
whff_status_t whff_gemv_plan_destroy(whff_gemv_plan_t plan);

/* ------------------------------------------------------------------ */
/* Dense GEMV: the plugin's gemv_kernel (K:80-132)                       */
/* ------------------------------------------------------------------ */

whff_status_t whff_gemv_workspace_size(uint64_t rows, uint64_t cols, int policy, int shape,
                                       int fanout, size_t* bytes);
/* y[i] = sum_j A[i*lda + j] * v[j]; policy/shape/fanout as K:80-84.      */
whff_status_t whff_gemv(const float* a_dev, uint64_t lda, uint64_t rows, uint64_t cols,
                        const float* v_dev, float* y_dev, int policy, int shape, int fanout,
                        void* workspace_dev, size_t workspace_bytes, whff_stream_t stream);
/* binary64 ground truth (mpgemv.py:64-69 gemv_oracle): y64 = cumsum order */
whff_status_t whff_gemv_oracle(const float* a_dev, uint64_t lda, uint64_t rows, uint64_t cols,
                               const float* v_dev, double* y_dev, whff_stream_t stream);
/* The same on binary64 inputs (mpgemv.py:64-69 casts to float64 first:
 * binary64 products, sequential sum).                                     */
whff_status_t whff_gemv_oracle_f64(const double* A, uint64_t lda, uint64_t rows, uint64_t cols,
                                   const double* v, double* y, whff_stream_t stream);

/* First non-finite element (mpgemv.py:42-51, codec.py:231, thermal.py:91-95):
 * atomically lowers *status_dev to its flat index.                       */
whff_status_t whff_find_nonfinite(const float* x_dev, uint64_t n, uint64_t* status_dev,
                                  whff_stream_t stream);

/* ------------------------------------------------------------------ */
/* Thermal model (thermal.py:81-117)                                     */
/* ------------------------------------------------------------------ */

/* y = fp32(A64 x + diag(b) u): thermal.py:98-109 when b/u are given,
 * thermal.py:112-117 (interpolation) when b_dev == u_dev == NULL.
 * CSR with binary64 values accumulated in CSR order (scipy csr_matvec).  */
whff_status_t whff_csr_matvec(const int64_t* indptr_dev, const int32_t* indices_dev,
                              const double* data_dev, uint64_t n_rows, const float* x_dev,
                              const float* b_dev, const float* u_dev, float* y_dev,
                              whff_stream_t stream);
/* u = fp32(fp32(dose) * footprint + dark) (thermal.py:81-88); footprint
 * NULL = dark step (u = dark).                                           */
whff_status_t whff_source_term(const float* footprint_dev, const float* dark_dev, float dose,
                               uint64_t n, float* u_dev, whff_stream_t stream);

/* ------------------------------------------------------------------ */
/* Device clock for the real-time scan (pipeline.py:164-289, 290-345)   */
/* ------------------------------------------------------------------ */

/* *t_dev = the device's %globaltimer (ns), written in stream order.       */
whff_status_t whff_device_timestamp(uint64_t* t_dev, whff_stream_t stream);
/* Holds the stream until %globaltimer >= *base_dev + offset_ns: paces the
 * schedule's millisecond steps on the device (replaces the reference's
 * simulated clock / wall-clock producer thread).                          */
whff_status_t whff_wait_until(const uint64_t* base_dev, uint64_t offset_ns, whff_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* WHFF_B200_H */
