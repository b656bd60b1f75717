/*
 * embc_cuda.h -- C ABI of the B200-native embedding-lookup codec
 * (libembc_cuda.so, built for sm_100a from paper_2407_04272_b200/csrc).
 *
 * This is the drop-in boundary for the reference's C++ codec API
 * (/root/reference/proj/include/embc/, namespace embc).  Every entry point
 * names the reference interface it replaces.  The reference has no FFI of its
 * own (it is header-only C++20); INTEGRATION.md shows the C++ call sites a
 * maintainer rewires, and include/embc_b200.hpp is the header-only C++
 * wrapper with the reference's types, names and exception classes.
 *
 * Conventions
 *   - Plain pointers and sizes only.  "d_" pointers are device memory, "h_"
 *     pointers host memory.  The caller owns every buffer.
 *   - Launches are asynchronous on the caller's stream (a cudaStream_t passed
 *     as void*; NULL = legacy default stream).  Data-dependent failures
 *     (non-finite values, malformed streams, ...) are recorded on the device
 *     and surface at the next embc_sync(), which returns the failure's status
 *     and fills embc_get_error() with the reference's exception text.
 *   - No exceptions cross the ABI.  EMBC_OK == 0.
 *   - Identical inputs give byte-identical outputs regardless of stream,
 *     grid shape or run (offsets are scan-derived, never atomics-ordered).
 */
#ifndef EMBC_CUDA_H_
#define EMBC_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EMBC_ABI_VERSION 1

typedef struct embc_ctx embc_ctx;

/* Status codes: the reference's exception classes (errors.hpp:24-45) plus
 * the failure modes a device library adds. */
typedef enum {
  EMBC_OK = 0,
  EMBC_ERR_VALUE = 1,       /* embc::ValueError  (errors.hpp:30-33) */
  EMBC_ERR_FORMAT = 2,      /* embc::FormatError (errors.hpp:36-39) */
  EMBC_ERR_CONFIG = 3,      /* embc::ConfigError (errors.hpp:42-45) */
  EMBC_ERR_CUDA = 4,        /* CUDA runtime failure */
  EMBC_ERR_CAPACITY = 5,    /* caller buffer too small */
  EMBC_ERR_ARGUMENT = 6,    /* null pointer / bad enum at the ABI */
  EMBC_ERR_UNSUPPORTED = 7, /* input outside the GPU path's supported envelope */
  EMBC_ERR_NCCL = 8         /* NCCL failure in the exchange */
} embc_status;

/* Codec tags == embc::Codec (container.hpp:32-36). */
enum { EMBC_CODEC_RAW = 0, EMBC_CODEC_VLZ = 1, EMBC_CODEC_HUFFMAN = 2 };

/* Encode output layouts. */
enum {
  EMBC_LAYOUT_CHUNKS = 0,  /* serialize_chunk() bodies back to back        (container.hpp:74-85) */
  EMBC_LAYOUT_PACKED = 1,  /* PackedSendBuffer: pack(chunks)               (container.hpp:242-256) */
  EMBC_LAYOUT_PAYLOAD = 2  /* codec payloads only (vlz tokens / huffman stream / raw u32le) */
};

/* Job input kinds. */
enum {
  EMBC_SRC_F32 = 0,  /* fp32 embedding values, quantized on the fly */
  EMBC_SRC_I32 = 1   /* int32 quantization codes (QuantizedBatch.codes) */
};

/* Failure reason codes (the reference throw sites). */
enum {
  EMBC_R_NONE = 0,
  EMBC_R_NONFINITE = 1,       /* quantizer.hpp:44-46   "non-finite value at index N" */
  EMBC_R_OVERFLOW = 2,        /* quantizer.hpp:50-53/:71-74 "quantization code overflow at index N..." */
  EMBC_R_EB_TOO_SMALL = 3,    /* quantizer.hpp:65-68   "error bound E too small ... at index N" */
  EMBC_R_BAD_WINDOW = 4,      /* vlz.hpp:39-43 */
  EMBC_R_TRUNCATED = 5,       /* bytes.hpp:157-162 */
  EMBC_R_VARINT_LONG = 6,     /* bytes.hpp:146 */
  EMBC_R_VLZ_DIM0 = 7,        /* vlz.hpp:131 */
  EMBC_R_VLZ_BAD_OFFSET = 8,  /* vlz.hpp:142-145 */
  EMBC_R_VLZ_BAD_TAG = 9,     /* vlz.hpp:148-151 */
  EMBC_R_VLZ_TRAILING = 10,   /* vlz.hpp:153-156 */
  EMBC_R_HUF_EMPTY = 11,      /* huffman.hpp:229 */
  EMBC_R_HUF_LEN_CAP = 12,    /* huffman.hpp:112-115 */
  EMBC_R_HUF_EMPTY_BOOK = 13, /* huffman.hpp:133 */
  EMBC_R_HUF_LEN_RANGE = 14,  /* huffman.hpp:138-140 */
  EMBC_R_HUF_KRAFT = 15,      /* huffman.hpp:143-145 */
  EMBC_R_HUF_PREFIX = 16,     /* huffman.hpp:175-177 */
  EMBC_R_HUF_DUP = 17,        /* huffman.hpp:183-185 */
  EMBC_R_HUF_EXHAUSTED = 18,  /* bitstream.hpp:65-67 */
  EMBC_R_HUF_BAD_CODE = 19,   /* huffman.hpp:285-287 */
  EMBC_R_BAD_MAGIC = 20,      /* container.hpp:91-93 */
  EMBC_R_BAD_VERSION = 21,    /* container.hpp:96-98 */
  EMBC_R_BAD_CODEC = 22,      /* container.hpp:100-102 */
  EMBC_R_PAYLEN = 23,         /* container.hpp:108-111 */
  EMBC_R_BAD_EB = 24,         /* batch.hpp:33-37 */
  EMBC_R_RAW_SIZE = 25,       /* container.hpp:152-155 */
  EMBC_R_HUF_COUNT = 26,      /* container.hpp:169-172 */
  EMBC_R_DIM0 = 27,           /* batch.hpp:72 */
  EMBC_R_PACK_OFFSET = 28,    /* container.hpp:271-275 */
  EMBC_R_PACK_OVERRUN = 29,   /* container.hpp:276-278 */
  EMBC_R_PACK_TRAILING = 30,  /* container.hpp:281-284 */
  EMBC_R_CAPACITY = 31,       /* output larger than the caller's capacity */
  EMBC_R_META_MISMATCH = 32,  /* commsim.hpp:371-376 metadata disagrees with chunk */
  EMBC_R_RANGE = 33           /* huffman alphabet span beyond the GPU histogram (EMBC_ERR_UNSUPPORTED) */
};

typedef struct {
  int32_t status;  /* embc_status of the first failure */
  int32_t reason;  /* EMBC_R_* */
  uint32_t job;    /* job / chunk index (lowest failing one) */
  uint32_t pad;
  uint64_t index;  /* element / token / symbol index inside that job */
  uint64_t a, b;   /* reason payload (lengths, offsets, tags, depths) */
  char message[320]; /* the reference's what() text for this failure */
} embc_error;

/* One compression unit: the reference's EncodeJob (container.hpp:295-300)
 * with the EmbeddingBatch replaced by a device tensor. */
typedef struct {
  const void* src;    /* device: n*dim fp32 values (EMBC_SRC_F32) or int32 codes (EMBC_SRC_I32) */
  uint32_t dim;       /* vector length (EmbeddingBatch::dim) */
  uint32_t n;         /* vector count */
  double eb;          /* absolute error bound (ErrorBound::value) */
  uint32_t window;    /* VlzConfig::window, [1, 65536] (vlz.hpp:36-46) */
  uint8_t codec;      /* EMBC_CODEC_* */
  uint8_t src_kind;   /* EMBC_SRC_* */
  uint8_t pad[2];
} embc_job;

/* One chunk to decode.  Shape/codec come from the metadata round
 * (ChunkMetadata, container.hpp:186-194) so launches need no device->host
 * read; the device verifies the chunk header against them. */
typedef struct {
  uint64_t offset;   /* byte offset of the serialized chunk (or payload) in d_in */
  uint64_t length;   /* serialized length (ChunkMetadata::compressed_len) */
  void* out;         /* device output: count*dim float, double or int32 */
  uint32_t dim;      /* expected ChunkMetadata::dim */
  uint32_t count;    /* expected ChunkMetadata::vector_count */
  double eb;         /* payload-only decode: error bound (ignored when a header is present) */
  uint8_t codec;     /* expected codec */
  uint8_t pad[7];
} embc_chunk_ref;

/* Decode output element types. */
enum { EMBC_OUT_F32 = 0, EMBC_OUT_F64 = 1, EMBC_OUT_I32_CODES = 2 };

/* ---- context --------------------------------------------------------- */

/* One context per (device, host thread).  It owns the codec scratch and
 * the device-side error record.  Replaces nothing in the reference (which is
 * allocation-per-call); needed so launches are graph-capturable. */
embc_status embc_ctx_create(int device, embc_ctx** out);
void embc_ctx_destroy(embc_ctx* ctx);

/* Pre-size scratch for up to `max_jobs` jobs / `max_values` values /
 * `max_tiles` tiles so later launches allocate nothing (required before CUDA
 * graph capture). */
embc_status embc_reserve(embc_ctx* ctx, uint32_t max_jobs, uint64_t max_values,
                         uint64_t max_payload_bytes);

/* CUDA-graph capture support: calls made while `stream` is capturing take
 * their descriptor staging from a pinned arena of `bytes` that stays valid
 * for the graphs' lifetime (reserve before capturing; embc_capture_reset
 * recycles it once those graphs are destroyed). */
embc_status embc_reserve_capture(embc_ctx* ctx, uint64_t bytes);
embc_status embc_capture_reset(embc_ctx* ctx);

/* Per-kernel CUDA-event timing on the launching stream.  While enabled, every
 * kernel launch is bracketed by events; embc_timing_collect() synchronises
 * the stream and returns (name, ms) pairs: names NUL-separated in `names`.
 * Returns the number of entries (or -1). */
embc_status embc_timing_enable(embc_ctx* ctx, int on);
int embc_timing_collect(embc_ctx* ctx, void* stream, char* names, size_t names_cap, float* ms,
                        int max_entries);

/* Waits for `stream`, then folds any device-recorded failure into the
 * context.  Returns that failure's status (or EMBC_OK) and clears it. */
embc_status embc_sync(embc_ctx* ctx, void* stream);

/* Copies the last failure (from any call) into *out. */
embc_status embc_get_error(const embc_ctx* ctx, embc_error* out);

/* Library version / build info ("embc_cuda <ver> sm_100a"). */
const char* embc_version(void);

/* ---- compression (container.hpp:119-142, :242-256, :294-311) ---------- */

/* Upper bound on the bytes embc_encode() can produce for these jobs. */
uint64_t embc_encode_bound(const embc_job* h_jobs, uint32_t njobs, int layout);

/* encode_chunks(jobs) followed by serialize_chunk() or pack(): quantize,
 * dedup / entropy-code, and lay every job's chunk out contiguously in job
 * order starting at d_out.
 *   d_offsets[j], d_lengths[j]  (device u64, may be NULL) chunk placement
 *   d_meta      (device, 25*njobs bytes, may be NULL) serialize_metadata()
 *               records (container.hpp:196-209)
 *   d_total     (device u64, may be NULL) total bytes written
 * Replaces embc::encode_chunks + embc::pack (container.hpp:304-311, :242-256)
 * and embc::encode_chunk + serialize_chunk for njobs == 1. */
embc_status embc_encode(embc_ctx* ctx, const embc_job* h_jobs, uint32_t njobs, int layout,
                        uint8_t* d_out, uint64_t cap, uint64_t* d_offsets, uint64_t* d_lengths,
                        uint8_t* d_meta, uint64_t* d_total, void* stream);

/* ---- decompression (container.hpp:89-115, :146-181) -------------------- */

/* parse_chunk() + decode_chunk() for each ref; outputs written as
 * out_kind (fp32 = float(reference double), fp64 = reference bits, or the
 * raw int32 codes).  With payload_only != 0 the refs point at bare codec
 * payloads (vlz_decode / huff_decode on codes). */
embc_status embc_decode(embc_ctx* ctx, const uint8_t* d_in, const embc_chunk_ref* h_refs,
                        uint32_t nrefs, int out_kind, int payload_only, void* stream);

/* embc_decode with the chunk lengths (and offsets) in DEVICE memory, as they
 * arrive from a peer: h_refs[c].offset is the chunk's base offset in d_in and
 * h_refs[c].length its capacity (the most bytes its sender may write); the
 * chunk is d_len[c] bytes at d_in + h_refs[c].offset + (d_off ? d_off[c] : 0).
 * The decode plan is computed on the device, so the call needs no host read
 * and can be captured in a CUDA graph.  A length above the capacity fails the
 * chunk (EMBC_ERR_FORMAT, reason EMBC_R_CAPACITY).  Replaces the receiving
 * half of Simulator::rank_body stage 4 (commsim.hpp:356-378) without the
 * metadata round trip through the host. */
embc_status embc_decode_dev(embc_ctx* ctx, const uint8_t* d_in, const embc_chunk_ref* h_refs, uint32_t nrefs,
                            const uint64_t* d_off, const uint64_t* d_len, int out_kind, int payload_only,
                            void* stream);

/* Number of chunks of the last embc_decode call that took the exact
 * sequential walker instead of the parallel decoders (malformed input, or a
 * shape outside the parallel envelope).  Synchronous. */
embc_status embc_decode_fallbacks(embc_ctx* ctx, uint32_t* h_count);

/* ---- building blocks exposed for parity tests and the analysis path ---- */

/* quantize() (quantizer.hpp:83-91) of fp32 (x_f64 == 0) or fp64 values. */
embc_status embc_quantize(embc_ctx* ctx, const void* d_x, int x_f64, uint64_t n, double eb,
                          int32_t* d_codes, void* stream);

/* dequantize() (quantizer.hpp:95-102) to fp32 or fp64. */
embc_status embc_dequantize(embc_ctx* ctx, const int32_t* d_codes, uint64_t n, double eb,
                            void* d_out, int out_f64, void* stream);

/* match_stats() (vlz.hpp:162-168) on int32 codes; results to host after sync. */
embc_status embc_match_stats(embc_ctx* ctx, const int32_t* d_codes, uint32_t dim, uint32_t n,
                             uint32_t window, uint64_t* h_literals, uint64_t* h_references,
                             void* stream);

/* detail::pattern_counts() (policy.hpp:167-173): distinct value rows and
 * distinct code rows of an fp32 sample; results to host after sync. */
embc_status embc_pattern_counts(embc_ctx* ctx, const float* d_x, uint32_t dim, uint32_t rows,
                                double eb, uint64_t* h_original, uint64_t* h_quantized,
                                void* stream);

/* ---- compressed embedding all-to-all over NCCL ---------------------------
 *
 * Replaces the reference's in-process exchange, Simulator::rank_body stages
 * 1-4 (commsim.hpp:286-435), with a real one between the GPUs of a node: one
 * process per GPU, one exchange object per process.  Table t is owned by rank
 * t mod R.
 *   forward : the owner's [R*B, dim] lookup output of table t is cut into R
 *             [B, dim] chunks, chunk d goes to rank d;
 *   backward: every rank's [B, dim] gradient slice of table t goes to its
 *             owner, which receives [R*B, dim] (rows s*B.. from rank s).
 * Each direction: compress the rank's (destination, table) chunks (one
 * embc_encode per table group), exchange the 25-byte ChunkMetadata records
 * (container.hpp:186-221; commsim.hpp:321-330), exchange the payloads with
 * grouped ncclSend/ncclRecv, decode every received chunk straight into the
 * caller's tensors on a decode stream.  With groups > 1 the owned tables are
 * cut into groups so compression, transfer and decompression of successive
 * groups overlap.  The call returns when the outputs are complete on `stream`
 * (one host wait per group for the metadata: NCCL takes host byte counts).
 * Per-iteration bounds/codecs come from the host controller (eb_at,
 * policy.hpp:336-342). */
typedef struct embc_exchange embc_exchange;

typedef struct {
  uint64_t uncompressed_bytes; /* fp32 bytes of chunks sent to other ranks (commsim.hpp:351-353) */
  uint64_t payload_bytes;      /* serialized chunk bytes sent to other ranks (commsim.hpp:326-328) */
  uint64_t metadata_bytes;     /* 25 B per chunk sent to another rank */
  uint64_t sent_values;        /* values compressed (all chunks, own rank included) */
  uint64_t sent_bytes;         /* serialized bytes of all compressed chunks */
  uint64_t recv_values;        /* values decoded */
  uint64_t recv_bytes;         /* serialized bytes of all decoded chunks */
} embc_exchange_stats;

/* ncclGetUniqueId(): rank 0 creates it and shares it with the other ranks. */
embc_status embc_exchange_unique_id(uint8_t out[128]);
/* One exchange per (process, GPU): an NCCL communicator of `nranks` ranks,
 * codec contexts for compression and decompression, and its streams. */
embc_status embc_exchange_create(int device, int rank, int nranks, const uint8_t id[128],
                                 uint32_t groups, embc_exchange** out);
void embc_exchange_destroy(embc_exchange* ex);
embc_status embc_exchange_get_error(const embc_exchange* ex, embc_error* out);

/* Forward: d_lookups[t] ([R*batch, dim] fp32) for the tables this rank owns
 * (others ignored), ebs[t] / codecs[t] for every table; d_outs[t] ([batch,
 * dim] fp32) for every table receive this rank's slice. */
embc_status embc_exchange_fwd(embc_exchange* ex, uint32_t ntables, uint32_t dim, uint32_t batch,
                              const float* const* d_lookups, const double* ebs,
                              const uint8_t* codecs, uint32_t window, float* const* d_outs,
                              embc_exchange_stats* stats, void* stream);
/* Backward: d_grads[t] ([batch, dim]) for every table; d_outs[t] ([R*batch,
 * dim]) for the tables this rank owns. */
embc_status embc_exchange_bwd(embc_exchange* ex, uint32_t ntables, uint32_t dim, uint32_t batch,
                              const float* const* d_grads, const double* ebs,
                              const uint8_t* codecs, uint32_t window, float* const* d_outs,
                              embc_exchange_stats* stats, void* stream);
/* The uncompressed baseline: the same tensors as raw fp32 grouped
 * ncclSend/ncclRecv (commsim.hpp:331-347, :380-397). */
embc_status embc_exchange_baseline_fwd(embc_exchange* ex, uint32_t ntables, uint32_t dim,
                                       uint32_t batch, const float* const* d_lookups,
                                       float* const* d_outs, void* stream);
embc_status embc_exchange_baseline_bwd(embc_exchange* ex, uint32_t ntables, uint32_t dim,
                                       uint32_t batch, const float* const* d_grads,
                                       float* const* d_outs, void* stream);

/* Transport of the exchange: 0 = NCCL (a 25-B metadata round, the byte
 * counts to the host, a variable-size payload round); 1 = peer-to-peer
 * windows: each rank's encode kernels write its chunks, lengths and offsets
 * straight into the destination's CUDA-IPC-shared window over NVLink, a
 * release flag per (source, destination) follows, and the destination waits
 * on the flags and decodes with embc_decode_dev -- no metadata round, no host
 * synchronisation, graph-capturable (the fused exchange of SURVEY.md 8(f)
 * row 1; the paper's future work).  Stats are filled only when
 * requested (that read synchronises). */
embc_status embc_exchange_set_mode(embc_exchange* ex, int mode);
/* Waits for the exchange's streams; reports a codec failure or a peer that
 * never signalled (mode 1, ~10 s) with the reference's rank/stage text. */
embc_status embc_exchange_sync(embc_exchange* ex);
/* embc_reserve_capture for both of the exchange's codec contexts (before
 * capturing embc_exchange_fwd / _bwd in a CUDA graph, mode 1). */
embc_status embc_exchange_reserve_capture(embc_exchange* ex, uint64_t bytes);

/* Per-kernel CUDA-event timing of the exchange's codec launches (both
 * contexts), as embc_timing_enable / embc_timing_collect. */
embc_status embc_exchange_timing_enable(embc_exchange* ex, int on);
int embc_exchange_timing_collect(embc_exchange* ex, char* names, size_t names_cap, float* ms,
                                 int max_entries);

/* ---- packed send buffer (container.hpp:258-292) --------------------------- */

/* unpack()'s validation of a PackedSendBuffer (host bytes): offsets start at
 * 4 + 16R and are contiguous, no entry runs past the end, no trailing bytes.
 * Writes up to `cap` (offset, length) pairs and the entry count.  The chunk
 * bodies are parsed by embc_decode on the device. */
embc_status embc_unpack(const uint8_t* h_buf, uint64_t len, uint64_t* h_offsets,
                        uint64_t* h_lengths, uint32_t cap, uint32_t* h_count, embc_error* err);

/* ---- host controller (policy.hpp), identical arithmetic ---------------- */

/* decay_multiplier() (policy.hpp:308-331); fn 0 stepwise, 1 linear, 2 log. */
embc_status embc_decay_multiplier(uint64_t iteration, int fn, double start_scale,
                                  uint64_t decay_end, uint32_t step_count, double* out);
/* classify_table() + PolicyConfig::eb_for() (policy.hpp:188-193, :95-102);
 * class 0 large, 1 medium, 2 small. */
embc_status embc_classify_table(double survival, double global_eb, double alpha, double beta,
                                double large_thr, double small_thr, int* cls, double* eb);
/* estimate_speedup() Eq. 2 (policy.hpp:202-208). */
embc_status embc_estimate_speedup(double ratio, double bandwidth, double comp_bps,
                                  double decomp_bps, double* out);

/* ---- synthetic workload (datagen.hpp), bit-identical to the reference -- */

/* gen_table() (datagen.hpp:115-126) rounded to fp32. dist 0 gaussian, 1 uniform. */
embc_status embc_gen_table(uint32_t rows, uint32_t dim, int dist, double mu, double sigma,
                           double lo, double hi, uint64_t seed, float* h_out);
/* gen_lookup_indices() (datagen.hpp:130-142, :89-110). */
embc_status embc_gen_lookup_indices(uint32_t rows, double zipf_s, uint64_t seed,
                                    uint32_t batch, uint64_t stream_id, uint32_t* h_out);
/* detail::mix_seed() (datagen.hpp:70-72). */
uint64_t embc_mix_seed(uint64_t seed, uint64_t salt);
/* Device gather: out[i, :] = table[idx[i], :] (Table::gather, datagen.hpp:158-166). */
embc_status embc_gather_rows(const float* d_table, uint32_t dim, const uint32_t* d_idx,
                             uint32_t batch, float* d_out, void* stream);

/* ---- simulator (commsim.hpp) with the codec on the GPU ------------------ */

/* TableSpec (datagen.hpp:36-47); table_id and seed are derived per rank. */
typedef struct {
  uint32_t rows, dim;
  int32_t dist;  /* 0 gaussian, 1 uniform */
  uint32_t pad;
  double mu, sigma, lo, hi, zipf_s;
} embc_sim_table;

/* SimConfig (commsim.hpp:30-62): the fields that enter the byte accounting. */
typedef struct {
  uint32_t ranks, batch, iterations, compression;
  uint64_t seed;
  double global_eb;
  int32_t decay_fn;  /* 0 stepwise, 1 linear, 2 log (policy.hpp:52-70) */
  uint32_t decay_steps;
  double decay_start_scale;
  uint64_t decay_end;
} embc_sim_config;

/* IterationStats (commsim.hpp:77-96); times are device-measured seconds. */
typedef struct {
  uint64_t iteration;
  double eb_max;
  uint64_t uncompressed_bytes, payload_bytes, metadata_bytes, wire_bytes;
  double comp_time, decomp_time, max_abs_error;
  uint64_t delivery_conserved, delivered_digest;
} embc_sim_iteration;

/* Simulator::run_schedule (commsim.hpp:253-266) + run_forward_alltoall
 * (:229-250): every rank compresses its table's per-destination batches with
 * embc_encode (packed), every received chunk is unpacked, checked against its
 * metadata and decoded with embc_decode into doubles.  prof_codec / prof_eb
 * are the TableProfile of table id r (= rank r), r < ranks.  Writes
 * `iterations` records and SimReport::deterministic_digest (:146-163). */
embc_status embc_simulate(int device, const embc_sim_config* cfg, const embc_sim_table* tables,
                          uint32_t ntables, const uint8_t* prof_codec, const double* prof_eb,
                          embc_sim_iteration* out, uint64_t* report_digest, embc_error* err);

#ifdef __cplusplus
}
#endif

#endif /* EMBC_CUDA_H_ */
