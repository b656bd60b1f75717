// embc_internal.h -- host-side structures shared by the encode/decode launch
// planners and the C ABI (not part of the public boundary).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/embc_cuda.h"
#include "embc_device.cuh"

namespace embc_dev {

// Per-job device descriptor for the encode pipeline.
struct DJob {
  const void* src;
  uint64_t N;         // values = dim * n
  uint64_t row_base;  // first global row index (per-row scratch arrays)
  uint32_t dim, n, window;
  uint32_t tile0, ntiles;
  uint32_t tile_rows;
  int32_t hjob;       // index among huffman jobs, -1 otherwise
  uint32_t header;    // 30 (chunks / packed layouts) or 0 (payload layout)
  uint8_t codec, src_kind, window_ok, pad;
  QParams qp;
  FastDiv fd;         // division by dim
  uint64_t hist_cap;  // huffman: bound on distinct symbols (min(N, kHistCap))
};

struct DTile {
  uint32_t job;
  uint32_t row0;  // first row inside the job
  uint32_t rows;
  uint32_t pad;
};

// Per-job mutable state (reset at the start of each call).
struct JobState {
  int32_t cmin, cmax;
  unsigned long long err;  // min err_key
  uint64_t payload;        // payload bytes
  uint64_t chunk_off;      // offset of the serialized chunk in d_out
  uint64_t bits;           // huffman payload bits
  uint32_t nsym;           // huffman distinct symbols
  uint32_t flags;
  uint64_t aux;            // reason payload (e.g. huffman depth)
  uint64_t lut_off;        // huffman: LUT entry of code cmin
  uint32_t wide;           // huffman: a code fell outside the speculative histogram window
  uint32_t tiles_done;     // emit: tiles of this job finished (last one merges edge bytes)
};

enum : uint32_t { JF_ABORT = 1u };

// Per-chunk decode descriptor (host-planned; shapes come from metadata).
// longest sleep between two polls of a flag another CTA of the launch sets (ns)
#ifndef EMBC_POLL_MAX_NS
#define EMBC_POLL_MAX_NS 256u
#endif
constexpr uint32_t kPollMaxNs = EMBC_POLL_MAX_NS;

struct DChunk {
  const uint8_t* in;   // start of the serialized chunk (or bare payload)
  uint64_t length;     // bytes of this chunk
  void* out;
  uint64_t N;          // dim * count
  uint32_t dim, count;
  double eb;           // payload-only: the caller's bound (else read from the header)
  uint8_t codec, payload_only, out_kind, seq;  // seq: decode with the exact sequential walker
  uint32_t book_cap;   // huffman: entry capacity
  FastDiv fd;          // division by dim
  // vlz plan
  uint32_t seg0, nseg;     // global segment index range
  uint64_t map_base;       // first segment-map entry
  uint64_t row_base;       // first per-row entry
  // huffman plan
  uint64_t tab_off;        // byte offset of this chunk's decode tables
  uint32_t nsub;           // 64-bit subsequences of the bitstream
  uint32_t blk0, nblk;     // global index range of this chunk's decode blocks
  uint8_t bad;             // device-planned calls: the received length exceeds the capacity
  uint8_t pad2[3];
};

// Per-chunk decode state (device).
struct DecState {
  unsigned long long err;  // (index << 6 | reason) of the first failure, ~0 = ok
  uint64_t a, b;
  double eb;               // parsed error bound
  uint64_t pay_off, pay_len;
  uint32_t nent, max_len;  // huffman codebook
  uint64_t nsym;           // huffman recorded symbol count
  uint64_t bit_off;        // huffman: bitstream offset inside the payload
};

}  // namespace embc_dev

// Context (opaque in the ABI).
struct embc_ctx {
  int device = 0;
  embc_error last{};
  // device memory
  embc_dev::DevError* d_err = nullptr;   // sticky error record (device)
  uint32_t* d_diag = nullptr;            // diagnostics of the last call (device)
  embc_dev::DevError* h_err = nullptr;   // pinned mirror
  uint8_t* d_scratch = nullptr;
  size_t scratch_cap = 0;
  // pinned descriptor staging: a ring of slots guarded by events, so an async
  // call never overwrites descriptors a previous call has not uploaded yet;
  // during CUDA-graph capture, slots come from a never-reused arena instead.
  static constexpr int kRing = 4;
  uint8_t* ring[kRing] = {};
  size_t ring_cap[kRing] = {};
  cudaEvent_t ring_evt[kRing] = {};
  int ring_next = 0;
  uint8_t* arena = nullptr;
  size_t arena_cap = 0, arena_used = 0;
  // device mirror of the capture arena: a captured call's descriptors go up
  // once at capture time, and the graph holds only a device-to-device copy
  // (a small pinned host-to-device copy node costs ~9 us per replay)
  uint8_t* darena = nullptr;
  cudaStream_t side = nullptr;  // non-blocking stream for those capture-time uploads
  // per-kernel CUDA-event timing (embc_timing_*)
  bool timing = false;
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> tev;
  std::vector<cudaEvent_t> ev_pool;
  uint8_t* d_hist = nullptr;             // huffman histograms (kept zero between calls)
  size_t hist_cap = 0;                   // entries
  // last call context for message formatting
  std::vector<double> job_eb;
  std::vector<uint32_t> job_window;
};

namespace embc_host {

cudaError_t ensure_scratch(embc_ctx* ctx, size_t bytes);
// Acquire `bytes` of pinned staging for one call on `stream`; call
// stage_commit after the cudaMemcpyAsync that reads it.
cudaError_t stage_acquire(embc_ctx* ctx, size_t bytes, cudaStream_t stream, uint8_t** out, int* slot);
cudaError_t stage_commit(embc_ctx* ctx, int slot, cudaStream_t stream);
// Upload `bytes` staged at `hs` (from stage_acquire) to device `dst` on
// `stream`, then commit the slot.
cudaError_t stage_upload(embc_ctx* ctx, void* dst, const uint8_t* hs, size_t bytes, int slot, cudaStream_t stream);
// Per-kernel timing hooks (no-ops unless embc_timing_enable(ctx, 1)).
void tmark_begin(embc_ctx* ctx, const char* name, cudaStream_t stream);
void tmark_end(embc_ctx* ctx, cudaStream_t stream);

#define EMBC_TIMED(ctx, name, stream, ...)   \
  do {                                       \
    embc_host::tmark_begin(ctx, name, stream); \
    __VA_ARGS__;                             \
    embc_host::tmark_end(ctx, stream);       \
  } while (0)
cudaError_t ensure_hist(embc_ctx* ctx, size_t entries);

embc_status set_error(embc_ctx* ctx, embc_status st, int reason, uint32_t job, uint64_t index,
                      uint64_t a, uint64_t b, const std::string& msg);
embc_status cuda_fail(embc_ctx* ctx, cudaError_t e, const char* where);
std::string format_message(int reason, uint64_t index, uint64_t a, uint64_t b, double eb);
std::string fmt_double(double v);  // std::to_string(double)

}  // namespace embc_host
