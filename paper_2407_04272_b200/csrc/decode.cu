// decode.cu -- sm_100a decompression in one launch: chunk parse/validation,
// raw / vlz / huffman decoding and dequantization straight into the consumer
// tensor.
//
// Mirrors embc::parse_chunk + embc::decode_chunk (container.hpp:89-115,
// :146-181), vlz_decode (vlz.hpp:129-158), huff_decode (huffman.hpp:254-291),
// dequantize (quantizer.hpp:95-102).
//
//   D1 k_dec_main   CTAs take work from an atomic ticket, in this order:
//     chunk CTAs    parse + validate every header (container.hpp:89-115); for
//                   huffman chunks also validate the codebook exactly as
//                   read_codebook + from_lengths + finalize and build the
//                   decode tables, then raise the chunk's ready flag.
//     vlz segments  2 KiB of tokens each: unit table, binary-lifting tables of
//                   the token chain, the segment's entry->exit map, a
//                   decoupled look-back over earlier segments for the true
//                   entry, then every token of the segment: literal rows
//                   decoded straight into the output, reference offsets
//                   validated (vlz.hpp:141-145).  The chunk's last segment to
//                   finish resolves reference chains to their root rows.
//     huffman blocks 8192 bits each: per 64-bit subsequence and entry offset
//                   the exit offset + symbol count (self-synchronising chains
//                   merged by codeword-start bitmaps), group/block maps, a
//                   decoupled look-back for the block's true entry, then the
//                   symbols, staged in shared memory and stored coalesced.
//     raw tiles     u32le -> values.
//     copy tiles    once a vlz chunk's segments are done: reference rows
//                   copied from their roots.
//     finishers     one per chunk, once its parallel decode is done: chunks
//                   the parallel path flagged (or planned sequential) are
//                   re-walked by the exact sequential decoders (the
//                   reference's first error and message); the last finisher
//                   folds the lowest failing chunk.
//   Later roles only ever wait on earlier tickets, so every wait is on a CTA
//   that is already resident or finished.
//
// Every malformed-input check of the reference is reproduced, in the
// reference's order, so the first failure (and its message) is identical.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "embc_internal.h"

namespace embc_dev {

// Rarely executed paths (sequential walkers, big-codebook tables, the error
// fold) and, optionally, the roles are kept out of line so the hot code of
// the roles resident on an SM stays compact in the instruction cache.
#ifndef EMBC_COLD
#define EMBC_COLD __device__ __noinline__
#endif
#ifndef EMBC_ROLE
#define EMBC_ROLE __device__
#endif

#include "decode_timeline.cuh"  // EMBC_DEBUG builds only: per-role device timestamps

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint32_t umin32(uint32_t a, uint32_t b) { return a < b ? a : b; }

__device__ __forceinline__ void dec_fail(DecState& S, uint64_t index, uint32_t reason, uint64_t a,
                                         uint64_t b) {
  if (S.err == ~0ull) {
    S.err = err_key(index, reason);
    S.a = a;
    S.b = b;
  }
}

// value of one decoded code in the requested output representation
__device__ __forceinline__ void store_value(const DChunk& C, uint64_t i, int32_t code, double w) {
  if (C.out_kind == EMBC_OUT_F32) {
    static_cast<float*>(C.out)[i] = __double2float_rn(reconstruct(code, w));
  } else if (C.out_kind == EMBC_OUT_F64) {
    static_cast<double*>(C.out)[i] = reconstruct(code, w);
  } else {
    static_cast<int32_t*>(C.out)[i] = code;
  }
}

__device__ __forceinline__ void copy_value(const DChunk& C, uint64_t dst, uint64_t src) {
  if (C.out_kind == EMBC_OUT_F64) {
    static_cast<double*>(C.out)[dst] = static_cast<double*>(C.out)[src];
  } else {
    static_cast<uint32_t*>(C.out)[dst] = static_cast<uint32_t*>(C.out)[src];
  }
}

// ---------------------------------------------------------------------------
// Header parse (container.hpp:89-115) + metadata agreement
// (commsim.hpp:371-376) + ErrorBound (container.hpp:147, batch.hpp:33-37)
// + raw size (container.hpp:152-155).  Deterministic: every CTA of a chunk
// computes the same state; the chunk CTA stores it.
// ---------------------------------------------------------------------------
__device__ DecState parse_chunk_hb(const DChunk& C, const uint8_t* hb);
__device__ DecState parse_chunk(const DChunk& C) {
  // the 30 header bytes in one round of independent loads, then parsed from registers
  uint8_t hb[kHeader];
  if (!C.payload_only) {
#pragma unroll
    for (uint32_t k = 0; k < kHeader; ++k) hb[k] = k < C.length ? __ldg(C.in + k) : 0;
  }
  return parse_chunk_hb(C, hb);
}
// parse_chunk on header bytes already at hand (hb[k] = byte k, 0 past the chunk)
__device__ DecState parse_chunk_hb(const DChunk& C, const uint8_t* hb) {
  DecState S;
  S.err = ~0ull;
  S.a = S.b = 0;
  S.eb = C.eb;
  S.pay_off = 0;
  S.pay_len = C.length;
  S.nent = S.max_len = 0;
  S.nsym = 0;
  S.bit_off = 0;
  if (!C.payload_only) {
    const uint8_t* p = hb;
    const uint64_t L = C.length;
    // field layout: magic[4] ver codec eb:8 dim:4 count:4 paylen:8
    const uint32_t need_at[] = {0, 1, 2, 3, 4, 5, 6, 14, 18, 22};
    const uint32_t need_n[] = {1, 1, 1, 1, 1, 1, 8, 4, 4, 8};
    const char magic[4] = {'E', 'M', 'B', 'C'};
    bool ok = true;
    for (int f = 0; f < 10 && ok; ++f) {
      const uint64_t at = need_at[f], k = need_n[f];
      if (L - at < k || L < at) {  // ByteReader::need (bytes.hpp:157-162)
        dec_fail(S, L - at, EMBC_R_TRUNCATED, k, at);
        ok = false;
        break;
      }
      if (f < 4 && p[f] != static_cast<uint8_t>(magic[f])) {
        dec_fail(S, 0, EMBC_R_BAD_MAGIC, 0, 0);
        ok = false;
      } else if (f == 4 && p[4] != 1) {
        dec_fail(S, 0, EMBC_R_BAD_VERSION, p[4], 0);
        ok = false;
      } else if (f == 5 && p[5] > 2) {
        dec_fail(S, 0, EMBC_R_BAD_CODEC, p[5], 0);
        ok = false;
      }
    }
    if (ok) {
      const uint64_t paylen = ld_le(p + 22, 8);
      if (paylen != L - kHeader) {
        dec_fail(S, 0, EMBC_R_PAYLEN, paylen, L - kHeader);
        ok = false;
      }
    }
    if (ok) {
      const uint32_t hdim = static_cast<uint32_t>(ld_le(p + 14, 4));
      const uint32_t hcount = static_cast<uint32_t>(ld_le(p + 18, 4));
      if (hcount != C.count || hdim != C.dim || p[5] != C.codec) {
        dec_fail(S, 0, EMBC_R_META_MISMATCH, hcount, C.count);
        ok = false;
      }
    }
    if (ok) {
      const uint64_t ebits = ld_le(p + 6, 8);
      double eb;
      memcpy(&eb, &ebits, 8);
      S.eb = eb;
      S.pay_off = kHeader;
      S.pay_len = L - kHeader;
    }
  }
  if (S.err == ~0ull && !(isfinite(S.eb) && S.eb > 0.0)) dec_fail(S, 0, EMBC_R_BAD_EB, 0, 0);
  if (S.err == ~0ull && C.codec == EMBC_CODEC_RAW && S.pay_len != 4 * C.N)
    dec_fail(S, 0, EMBC_R_RAW_SIZE, S.pay_len, C.N);
  return S;
}

// ---------------------------------------------------------------------------
// raw payload (container.hpp:151-160): u32le codes -> values
// ---------------------------------------------------------------------------
struct RawTile {
  uint32_t chunk;
  uint32_t pad;
  uint64_t e0, ne;
};

// 16 bytes at byte offset s (0..15, uniform) of the 32-byte window a|b, as four
// little-endian u32 words
__device__ __forceinline__ uint4 window16(const uint4 a, const uint4 b, uint32_t s) {
  const uint32_t m = s >> 2, r = 8 * (s & 3);
  const uint32_t w0 = m == 0 ? a.x : m == 1 ? a.y : m == 2 ? a.z : a.w;
  const uint32_t w1 = m == 0 ? a.y : m == 1 ? a.z : m == 2 ? a.w : b.x;
  const uint32_t w2 = m == 0 ? a.z : m == 1 ? a.w : m == 2 ? b.x : b.y;
  const uint32_t w3 = m == 0 ? a.w : m == 1 ? b.x : m == 2 ? b.y : b.z;
  const uint32_t w4 = m == 0 ? b.x : m == 1 ? b.y : m == 2 ? b.z : b.w;
  return make_uint4(__funnelshift_r(w0, w1, r), __funnelshift_r(w1, w2, r), __funnelshift_r(w2, w3, r),
                    __funnelshift_r(w3, w4, r));
}

// fp32 output, whole quads: aligned 16-B loads of the (unaligned) code words,
// 16-B stores, four quads in flight per thread
__device__ __forceinline__ void raw_tile_f32(const DChunk& C, const uint8_t* p, double w, const RawTile& T) {
  const uintptr_t g0 = reinterpret_cast<uintptr_t>(p + 4 * T.e0);
  const uint4* gv = reinterpret_cast<const uint4*>(g0 & ~uintptr_t(15));
  const uint32_t s = static_cast<uint32_t>(g0 & 15);
  const uint32_t nq = static_cast<uint32_t>(T.ne >> 2);
  float4* o = reinterpret_cast<float4*>(static_cast<float*>(C.out) + T.e0);
  for (uint32_t q0 = 0; q0 < nq; q0 += 4 * blockDim.x) {
    uint4 lo[4], hi[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t q = q0 + u * blockDim.x + threadIdx.x;
      if (q < nq) {
        lo[u] = __ldg(gv + q);
        hi[u] = s ? __ldg(gv + q + 1) : lo[u];  // the block holding the quad's last byte
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t q = q0 + u * blockDim.x + threadIdx.x;
      if (q < nq) {
        const uint4 c = window16(lo[u], hi[u], s);
        o[q] = make_float4(__double2float_rn(reconstruct(static_cast<int32_t>(c.x), w)),
                           __double2float_rn(reconstruct(static_cast<int32_t>(c.y), w)),
                           __double2float_rn(reconstruct(static_cast<int32_t>(c.z), w)),
                           __double2float_rn(reconstruct(static_cast<int32_t>(c.w), w)));
      }
    }
  }
  for (uint64_t i = T.e0 + 4ull * nq + threadIdx.x; i < T.e0 + T.ne; i += blockDim.x) {
    const uint8_t* q = p + 4 * i;
    const int32_t code = static_cast<int32_t>(static_cast<uint32_t>(q[0]) | (static_cast<uint32_t>(q[1]) << 8) |
                                              (static_cast<uint32_t>(q[2]) << 16) |
                                              (static_cast<uint32_t>(q[3]) << 24));
    static_cast<float*>(C.out)[i] = __double2float_rn(reconstruct(code, w));
  }
}

__device__ __forceinline__ void raw_tile(const DChunk& C, const DecState& S, const RawTile& T) {
  if (S.err != ~0ull) return;
  const uint8_t* p = C.in + S.pay_off;
  const double w = 2.0 * S.eb;
  if (C.out_kind == EMBC_OUT_F32 && (reinterpret_cast<uintptr_t>(C.out) & 15) == 0 && (T.e0 & 3) == 0) {
    raw_tile_f32(C, p, w, T);
    return;
  }
  for (uint64_t i = T.e0 + threadIdx.x; i < T.e0 + T.ne; i += blockDim.x) {
    const uint8_t* q = p + 4 * i;
    const int32_t code = static_cast<int32_t>(static_cast<uint32_t>(q[0]) | (static_cast<uint32_t>(q[1]) << 8) |
                                              (static_cast<uint32_t>(q[2]) << 16) |
                                              (static_cast<uint32_t>(q[3]) << 24));
    store_value(C, i, code, w);
  }
}

// ---------------------------------------------------------------------------
// D2: vlz token walk (vlz.hpp:129-158), exact reference semantics.
// One thread per chunk; also the error reproducer for the parallel decoder.
// ---------------------------------------------------------------------------
// ByteReader::varint (bytes.hpp:139-147): <= 10 bytes, bits beyond 64 dropped.
__device__ __forceinline__ bool rd_varint(const uint8_t* p, uint64_t L, uint64_t& pos, uint64_t& v,
                                          DecState& S, uint64_t) {
  v = 0;
  for (int shift = 0; shift < 64; shift += 7) {
    if (pos >= L) {
      dec_fail(S, L - pos, EMBC_R_TRUNCATED, 1, pos);
      return false;
    }
    const uint8_t b = p[pos++];
    v |= static_cast<uint64_t>(b & 0x7F) << shift;
    if (!(b & 0x80)) return true;
  }
  dec_fail(S, 0, EMBC_R_VARINT_LONG, pos, 0);
  return false;
}

EMBC_COLD void k_dec_vlz_seq_cta(uint32_t bid, const DChunk* __restrict__ ch, DecState* __restrict__ st,
                              const uint32_t* list, const volatile uint32_t* vflag) {
  if (threadIdx.x != 0) return;
  const uint32_t c = bid;
  const DChunk C = ch[c];
  DecState& S = st[c];
  if (S.err != ~0ull || !(C.seq || vflag[c])) return;  // only chunks the parallel path did not finish
  const uint8_t* p = C.in + S.pay_off;
  const uint64_t L = S.pay_len;
  const double w = 2.0 * S.eb;
  const uint32_t dim = C.dim, n = C.count;
  if (dim == 0 && n > 0) {
    dec_fail(S, 0, EMBC_R_VLZ_DIM0, 0, 0);
    return;
  }
  uint64_t pos = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (pos >= L) {
      dec_fail(S, L - pos, EMBC_R_TRUNCATED, 1, pos);
      return;
    }
    const uint8_t tag = p[pos++];
    if (tag == 0x00) {
      for (uint32_t j = 0; j < dim; ++j) {
        uint64_t v;
        if (!rd_varint(p, L, pos, v, S, i)) return;
        store_value(C, static_cast<uint64_t>(i) * dim + j, unzigzag(static_cast<uint32_t>(v)), w);
      }
    } else if (tag == 0x01) {
      uint64_t off;
      if (!rd_varint(p, L, pos, off, S, i)) return;
      if (off < 1 || off > i || off > kMaxWindow) {
        dec_fail(S, i, EMBC_R_VLZ_BAD_OFFSET, off, 0);
        return;
      }
      const uint64_t src = (static_cast<uint64_t>(i) - off) * dim;
      for (uint32_t j = 0; j < dim; ++j) copy_value(C, static_cast<uint64_t>(i) * dim + j, src + j);
    } else {
      dec_fail(S, i, EMBC_R_VLZ_BAD_TAG, tag, 0);
      return;
    }
  }
  if (pos != L) dec_fail(S, 0, EMBC_R_VLZ_TRAILING, L - pos, n);
}
// ===========================================================================
// Huffman: codebook tables (read_codebook + from_lengths + finalize,
// huffman.hpp:132-148, :165-186, :213-222), then a self-synchronising
// parallel decode of the MSB-first bitstream (huffman.hpp:254-291):
//   H0 k_huff_tables  per chunk: validate the codebook exactly as the
//                     reference does; canonical first/count/base per length, a
//                     2^11-entry prefix LUT and the per-entry output values.
//   H1 k_huff_spec    one thread per 256-bit subsequence decodes
//                     speculatively from the subsequence start to the first
//                     codeword boundary past its end.
//   H2 k_huff_sync    per chunk: re-decode subsequences whose true start (the
//                     predecessor's exit) differs until a fixpoint; scan the
//                     symbol counts into output offsets; check count/validity.
//   H3 k_huff_out     decode again from the true starts and write values.
// Failures flag the chunk; k_dec_huff_seq then reproduces the exact error.
// ===========================================================================
constexpr int kL0 = 10;
constexpr uint32_t kSubBits = 64;
constexpr uint32_t kLong = 63;

struct HTab {
  uint32_t first[33], count[33], base[33];
  uint32_t max_len, nent;
  uint64_t nsym, bit_off, nbits;
};

__host__ __device__ inline uint64_t htab_bytes(uint32_t cap) {
  return ((sizeof(HTab) + 4u * (1u << kL0) + 4ull * cap + 8ull * cap) + 15) & ~uint64_t(15);
}

struct HView {
  HTab* tab;
  uint32_t* lut;
  int32_t* syms;
  uint64_t* vals;
};

__device__ __forceinline__ HView hview(uint8_t* tabs, const DChunk& C) {
  HView v;
  uint8_t* b = tabs + C.tab_off;
  v.tab = reinterpret_cast<HTab*>(b);
  v.lut = reinterpret_cast<uint32_t*>(b + sizeof(HTab));
  v.syms = reinterpret_cast<int32_t*>(b + sizeof(HTab) + 4u * (1u << kL0));
  v.vals = reinterpret_cast<uint64_t*>(b + sizeof(HTab) + 4u * (1u << kL0) + 4ull * C.book_cap);
  return v;
}

__device__ void bitonic_sort_u64(uint64_t* key, uint32_t p2) {
  for (uint32_t k = 2; k <= p2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < p2; i += blockDim.x) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = key[i], b = key[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            key[i] = b;
            key[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ uint64_t value_bits(int32_t code, double w, int kind) {
  if (kind == EMBC_OUT_F32) return __float_as_uint(__double2float_rn(reconstruct(code, w)));
  if (kind == EMBC_OUT_F64) return static_cast<uint64_t>(__double_as_longlong(reconstruct(code, w)));
  return static_cast<uint32_t>(code);
}

// Codebook of <= 64 entries by one warp (two entries per lane): entry checks
// in entry order (huffman.hpp:137-141), Kraft (:143-148), canonical order
// (length, symbol) by rank counting over the staged keys, canonical codes
// (closed form of finalize, :165-181), duplicate symbols (:183-185).  Fills
// tb.first/base/count (zeroed by the caller), vals / syms (if given) and the
// left-aligned code starts.  Returns 0, or 1 length out of range (*bad =
// entry << 8 | length), 2 Kraft, 3 duplicate symbol.
__device__ int small_book_warp(const uint8_t* p, uint32_t nent, double w, int out_kind, HTab& tb, uint64_t* vals,
                               int32_t* syms, uint64_t* starts, uint64_t* kk, unsigned long long* bad_out) {
  const uint32_t lane = threadIdx.x & 31;
  uint64_t k[2];
  unsigned long long bad = ~0ull, kraft = 0;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const uint32_t i = r * 32 + lane;
    k[r] = ~0ull;
    if (i < nent) {
      const uint32_t sym = static_cast<uint32_t>(ld_be(p + 12 + 5 * i, 4));
      const uint32_t len = p[12 + 5 * i + 4];
      if (len == 0 || len > 32) bad = min(bad, (static_cast<unsigned long long>(i) << 8) | len);
      else kraft += 1ull << (32 - len);
      k[r] = (static_cast<uint64_t>(len) << 32) | (sym ^ 0x80000000u);
      kk[i] = k[r];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    kraft += __shfl_xor_sync(0xffffffffu, kraft, o);
  }
  if (bad != ~0ull) {
    *bad_out = bad;
    return 1;
  }
  if (kraft > (1ull << 32)) return 2;
  __syncwarp();
  // a codebook written by write_codebook is already in canonical order
  // (strictly ascending (length, symbol)): then the ranks are the entry
  // indices and only duplicate symbols need checking
  const uint64_t up0 = __shfl_up_sync(0xffffffffu, k[0], 1), up1 = __shfl_up_sync(0xffffffffu, k[1], 1);
  const uint64_t last0 = __shfl_sync(0xffffffffu, k[0], 31);
  bool srt = true;
  if (lane >= 1 && lane < nent) srt = up0 < k[0];
  if (32 + lane < nent) srt = srt && (lane == 0 ? last0 : up1) < k[1];
  if (__all_sync(0xffffffffu, srt)) {
    const uint32_t s0 = static_cast<uint32_t>(k[0]), s1 = static_cast<uint32_t>(k[1]);
    const bool v0 = lane < nent, v1 = 32 + lane < nent;
    // (warp collectives outside any short-circuit: every lane takes part)
    const uint32_t m0 = __match_any_sync(0xffffffffu, (static_cast<uint64_t>(v0) << 32) | s0);
    bool dup = v0 && __popc(m0) > 1;
    if (nent > 32) {
      const uint32_t m1 = __match_any_sync(0xffffffffu, (static_cast<uint64_t>(v1) << 32) | s1);
      dup |= v1 && __popc(m1) > 1;
      for (uint32_t j = 0; j < 32; ++j) {
        const uint32_t sj = __shfl_sync(0xffffffffu, s0, j);
        dup |= v1 && sj == s1;
      }
    }
    if (__any_sync(0xffffffffu, dup)) return 3;
  } else {
    uint32_t rank[2] = {0, 0};
    bool dup = false;
    for (uint32_t j = 0; j < nent; ++j) {
      const uint64_t kj = kk[j];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const uint32_t i = r * 32 + lane;
        rank[r] += (kj < k[r] || (kj == k[r] && j < i)) ? 1u : 0u;
        dup |= i < nent && j != i && static_cast<uint32_t>(kj) == static_cast<uint32_t>(k[r]);
      }
    }
    if (__any_sync(0xffffffffu, dup)) return 3;
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 2; ++r)
      if (r * 32 + lane < nent) kk[rank[r]] = k[r];
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 2; ++r) k[r] = r * 32 + lane < nent ? kk[r * 32 + lane] : ~0ull;
  }
  unsigned long long carry = 0;
  uint32_t prev_last = 0;  // length of the previous register's last element
  uint32_t maxl = 0;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const uint32_t i = r * 32 + lane;
    const bool v = i < nent;
    const uint32_t ln = v ? static_cast<uint32_t>(k[r] >> 32) : 0;
    maxl = max(maxl, ln);
    const unsigned long long kr = v ? (1ull << (32 - ln)) : 0;
    const unsigned long long inc = warp_incl_scan<unsigned long long>(kr);
    const uint32_t lp = __shfl_up_sync(0xffffffffu, ln, 1);
    const uint32_t lprev = lane ? lp : prev_last;
    if (v) {
      const uint32_t code = static_cast<uint32_t>((carry + inc - kr) >> (32 - ln));
      const uint32_t sy = static_cast<uint32_t>(k[r]) ^ 0x80000000u;
      if (i == 0 || lprev != ln) {
        tb.first[ln] = code;
        tb.base[ln] = i;
      }
      atomicAdd(&tb.count[ln], 1u);
      if (syms) syms[i] = static_cast<int32_t>(sy);
      vals[i] = value_bits(static_cast<int32_t>(sy), w, out_kind);
      starts[i] = (static_cast<uint64_t>(code) << (32 - ln)) | (static_cast<uint64_t>(ln) << 56);
    }
    carry += __shfl_sync(0xffffffffu, inc, 31);
    prev_last = __shfl_sync(0xffffffffu, ln, 31);
  }
  maxl = __reduce_max_sync(0xffffffffu, maxl);
  if (lane == 0) tb.max_len = maxl;
  return 0;
}

// Codebook of <= 64 entries: validation (huffman.hpp:132-148, entry order),
// canonical codes (finalize, :165-186), duplicate check (:183-185) by one warp
// (small_book_warp); the prefix LUT by the whole CTA.
__device__ void huff_tables_small(const DChunk& C, DecState& S, const uint8_t* p, uint64_t L, HView hv, HTab& tb,
                                  uint64_t* starts, uint32_t c, uint32_t* __restrict__ hflag) {
  __shared__ int s_stop2;
  const uint32_t nent = S.nent;
  if (threadIdx.x < 33) {
    tb.count[threadIdx.x] = 0;
    tb.first[threadIdx.x] = 0;
    tb.base[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) s_stop2 = 0;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned long long bad = 0;
    const int r = small_book_warp(p, nent, 2.0 * S.eb, C.out_kind, tb, hv.vals, hv.syms, starts, starts + 64, &bad);
    if (r && (threadIdx.x & 31) == 0) {
      if (r == 1) dec_fail(S, bad >> 8, EMBC_R_HUF_LEN_RANGE, bad & 0xFF, 0);
      else if (r == 2) dec_fail(S, 0, EMBC_R_HUF_KRAFT, 0, 0);
      else dec_fail(S, 0, EMBC_R_HUF_DUP, 0, 0);
      s_stop2 = 1;
    }
  }
  __syncthreads();
  DTS(8000 + c, 2);
  DTS(8000 + c, 3);
  DTS(8000 + c, 4);
  if (s_stop2) return;
  // left-aligned code starts ascending in canonical order -> prefix LUT
  for (uint32_t sl = threadIdx.x; sl < (1u << kL0); sl += blockDim.x) {
    const uint64_t V = static_cast<uint64_t>(sl) << (32 - kL0);
    const uint64_t Vend = V + (1ull << (32 - kL0));
    int lo = 0, hi = static_cast<int>(nent) - 1, f = -1;
    while (lo <= hi) {
      const int mid = (lo + hi) >> 1;
      if ((starts[mid] & 0xFFFFFFFFFFull) <= V) {
        f = mid;
        lo = mid + 1;
      } else {
        hi = mid - 1;
      }
    }
    uint32_t ent = 0;
    if (f >= 0) {
      const uint32_t ln = static_cast<uint32_t>(starts[f] >> 56);
      const uint64_t a0 = starts[f] & 0xFFFFFFFFFFull;
      if (V < a0 + (1ull << (32 - ln))) ent = ln <= kL0 ? (static_cast<uint32_t>(f) << 6) | ln : kLong;
    }
    if (!ent && f + 1 < static_cast<int>(nent) && (starts[f + 1] & 0xFFFFFFFFFFull) < Vend) ent = kLong;
    hv.lut[sl] = ent;
  }
  DTS(8000 + c, 5);
  DTS(8000 + c, 6);
  if (threadIdx.x == 0) {
    uint32_t max_len = 0;  // entries().back().length (huffman.hpp:257)
    for (uint32_t l = 1; l <= 32; ++l)
      if (tb.count[l]) max_len = l;
    tb.max_len = max_len;
    tb.nent = nent;
    tb.nsym = S.nsym;
    tb.bit_off = 12 + 5ull * nent;
    tb.nbits = 8 * (L - tb.bit_off);
    *hv.tab = tb;
    S.max_len = max_len;
    S.bit_off = tb.bit_off;
    if (S.nsym != C.N) hflag[c] = 1;  // decoded count != dim*count (container.hpp:169-172)
  }
}


// Block-local decode tables for a small codebook (<= 64 entries): a huffman
// block repeats the chunk CTA's checks and table build (huff_tables +
// huff_tables_small) on a shared-memory copy of the chunk's first bytes, so it
// need not wait for the chunk CTA.  Returns false when anything would differ
// from the plain path (any failure, a larger codebook, a count mismatch): the
// block then waits for the chunk CTA's verdict and tables.  Called by all
// threads; `hb` holds min(length, kLocalHdr) bytes of the chunk.
constexpr uint32_t kLocalHdr = kHeader + 12 + 5 * 64;
__device__ bool huff_tables_local(const DChunk& C, const uint8_t* hb, HTab& tb, uint32_t* lut, uint64_t* vals,
                                  uint64_t* starts) {
  __shared__ int s_ok;
  __shared__ uint32_t s_nent;
  __shared__ double s_w;
  if (threadIdx.x < 33) {
    tb.count[threadIdx.x] = 0;
    tb.first[threadIdx.x] = 0;
    tb.base[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) {
    // parse_chunk's checks, all passing (any failure: the chunk CTA decides)
    const uint64_t len = C.length;
    const uint32_t poff = C.payload_only ? 0 : kHeader;
    double eb = C.eb;
    bool ok = len >= poff;
    if (ok && !C.payload_only) {
      const uint64_t ebits = ld_le(hb + 6, 8);
      memcpy(&eb, &ebits, 8);
      ok = hb[0] == 'E' && hb[1] == 'M' && hb[2] == 'B' && hb[3] == 'C' && hb[4] == 1 && hb[5] == C.codec &&
           ld_le(hb + 22, 8) == len - kHeader && ld_le(hb + 14, 4) == C.dim && ld_le(hb + 18, 4) == C.count;
    }
    ok = ok && isfinite(eb) && eb > 0.0;
    const uint64_t L = len - poff;
    const uint8_t* p = hb + poff;
    uint64_t nent = 0;
    if (ok) ok = L >= 12 && poff + 12 <= kLocalHdr;
    if (ok) {
      nent = ld_be(p + 8, 4);
      ok = ld_be(p, 8) == C.N && nent >= 1 && nent <= 64 && nent <= (L - 12) / 5 && nent <= C.book_cap &&
           poff + 12 + 5 * nent <= kLocalHdr;
    }
    s_ok = ok;
    s_nent = static_cast<uint32_t>(nent);
    s_w = 2.0 * eb;
    if (ok) {
      tb.nent = static_cast<uint32_t>(nent);
      tb.nsym = C.N;
      tb.bit_off = 12 + 5ull * nent;
      tb.nbits = 8 * (L - tb.bit_off);
    }
  }
  __syncthreads();
  EMBC_DBG(const unsigned long long lt0 = dtime());
  if (!s_ok) return false;
  const uint32_t nent = s_nent;
  const uint8_t* p = hb + (C.payload_only ? 0 : kHeader);
  if (threadIdx.x < 32) {
    unsigned long long bad = 0;
    if (small_book_warp(p, nent, s_w, C.out_kind, tb, vals, nullptr, starts, starts + 64, &bad) && threadIdx.x == 0)
      s_ok = 0;
  }
  __syncthreads();
  EMBC_DBG(const unsigned long long lt1 = dtime());
  if (!s_ok) return false;
  // the prefix LUT straight from the canonical tables: a slot is the codeword
  // of length l <= kL0 whose code is its top l bits, else a prefix of a longer
  // codeword (kLong), else no codeword (0)
  //   Canonical codes of increasing length occupy increasing, contiguous
  //   slot ranges: length l holds [lim[l-1], lim[l]) with
  //   lim[l] = (first[l] + count[l]) << (kL0 - l); prefixes of longer codes
  //   follow up to lim[kL0 + 1]; an incomplete code leaves the rest empty.
  __shared__ uint32_t s_lim[kL0 + 2];
  const uint32_t ml = tb.max_len;
  if (threadIdx.x == 0) {
    uint32_t prev = 0;
    for (uint32_t l = 1; l <= kL0; ++l) {
      if (l <= ml && tb.count[l]) prev = (tb.first[l] + tb.count[l]) << (kL0 - l);
      s_lim[l] = prev;
    }
    uint32_t endl = prev;
    for (uint32_t l = kL0 + 1; l <= ml; ++l)
      if (tb.count[l])
        endl = max(endl, static_cast<uint32_t>(((static_cast<uint64_t>(tb.first[l]) + tb.count[l] - 1) >> (l - kL0)) + 1));
    s_lim[kL0 + 1] = endl;
  }
  __syncthreads();
  uint32_t lim[kL0 + 2];
#pragma unroll
  for (uint32_t l = 1; l <= kL0 + 1; ++l) lim[l] = s_lim[l];
  for (uint32_t sl = threadIdx.x; sl < (1u << kL0); sl += blockDim.x) {
    uint32_t ent = 0;
    if (sl < lim[kL0]) {
      uint32_t l = 1;
#pragma unroll
      for (uint32_t k = 1; k < kL0; ++k) l += sl >= lim[k] ? 1u : 0u;
      ent = ((tb.base[l] + (sl >> (kL0 - l)) - tb.first[l]) << 6) | l;
    } else if (sl < lim[kL0 + 1]) {
      ent = kLong;
    }
    lut[sl] = ent;
  }
  __syncthreads();
  EMBC_DBG(if (threadIdx.x == 0) {
    atomicAdd(&g_dloc[4], lt1 - lt0);
    atomicAdd(&g_dloc[5], dtime() - lt1);
  });
  return true;
}

EMBC_COLD void huff_tables(uint32_t c, const DChunk* __restrict__ ch, DecState& S,
                            uint64_t* __restrict__ keys, uint8_t* __restrict__ tabs,
                            uint32_t* __restrict__ hflag, uint64_t* skey, uint32_t skey_cap) {
  __shared__ unsigned long long s_tmp64[33];
  __shared__ unsigned long long s_bad;
  __shared__ int s_stop;
  __shared__ HTab tb;
  const DChunk C = ch[c];
  DTS(8000 + c, 8);
  if (S.err != ~0ull) return;
  const uint8_t* p = C.in + S.pay_off;
  const uint64_t L = S.pay_len;
  HView hv = hview(tabs, C);
  uint64_t* key = keys + (C.tab_off / 8);  // keys region mirrors the table offsets (sized >= p2)
  if (threadIdx.x == 0) {
    s_stop = 0;
    s_bad = ~0ull;
    // u64be symbol_count, u32be entry_count (huffman.hpp:214-215)
    if (L < 8) {
      dec_fail(S, L, EMBC_R_TRUNCATED, 8, 0);
      s_stop = 1;
    } else if (L < 12) {
      dec_fail(S, L - 8, EMBC_R_TRUNCATED, 4, 8);
      s_stop = 1;
    } else {
      S.nsym = ld_be(p, 8);
      const uint64_t nent = ld_be(p + 8, 4);
      const uint64_t fit = (L - 12) / 5;
      if (nent > fit) {  // first entry that does not fit
        const uint64_t at = 12 + 5 * fit;
        if (L - at < 4) dec_fail(S, L - at, EMBC_R_TRUNCATED, 4, at);
        else dec_fail(S, L - at - 4, EMBC_R_TRUNCATED, 1, at + 4);
        s_stop = 1;
      } else if (nent == 0) {
        dec_fail(S, 0, EMBC_R_HUF_EMPTY_BOOK, 0, 0);
        s_stop = 1;
      } else if (nent > C.book_cap) {
        dec_fail(S, 0, EMBC_R_RANGE, nent, C.book_cap);
        s_stop = 1;
      } else {
        S.nent = static_cast<uint32_t>(nent);
      }
    }
  }
  __syncthreads();
  if (s_stop) return;
  const uint32_t nent = S.nent;
  if (nent <= 64 && skey_cap >= 128) {  // small codebooks: one warp, the LUT by the CTA
    huff_tables_small(C, S, p, L, hv, tb, reinterpret_cast<uint64_t*>(skey), c, hflag);
    return;
  }
  // length range, in entry order (huffman.hpp:137-141), and Kraft sum
  unsigned long long kraft = 0;
  for (uint32_t i = threadIdx.x; i < nent; i += blockDim.x) {
    const uint8_t len = p[12 + 5ull * i + 4];
    if (len == 0 || len > 32) atomicMin(&s_bad, (static_cast<unsigned long long>(i) << 8) | len);
    else kraft += 1ull << (32 - len);
  }
  kraft = block_sum<unsigned long long>(kraft, s_tmp64);
  if (threadIdx.x == 0) {
    if (s_bad != ~0ull) {
      dec_fail(S, s_bad >> 8, EMBC_R_HUF_LEN_RANGE, s_bad & 0xFF, 0);
      s_stop = 1;
    } else if (kraft > (1ull << 32)) {
      dec_fail(S, 0, EMBC_R_HUF_KRAFT, 0, 0);
      s_stop = 1;
    }
  }
  __syncthreads();
  if (s_stop) return;
  // canonical order (length, symbol): key = len << 32 | (symbol ^ 0x80000000)
  uint32_t p2 = 1;
  while (p2 < nent) p2 <<= 1;
  uint32_t* ssym = nullptr;  // symbols in canonical order, kept in smem when there is room
  if (p2 + (p2 + 1) / 2 <= skey_cap) {
    key = skey;  // small codebooks sort in shared memory
    ssym = reinterpret_cast<uint32_t*>(skey + p2);
  }
  for (uint32_t i = threadIdx.x; i < p2; i += blockDim.x) {
    if (i < nent) {
      const uint32_t s = static_cast<uint32_t>(ld_be(p + 12 + 5ull * i, 4));
      key[i] = (static_cast<uint64_t>(p[12 + 5ull * i + 4]) << 32) | (s ^ 0x80000000u);
    } else {
      key[i] = ~0ull;
    }
  }
  __syncthreads();
  DTS(8000 + c, 2);
  if (ssym && p2 <= 256) {  // one warp, in registers
    if (threadIdx.x < 32) warp_sort_smem(key, p2);
    __syncthreads();
  } else {
    bitonic_sort_u64(key, p2);
  }
  DTS(8000 + c, 3);
  for (uint32_t i = threadIdx.x; i < nent; i += blockDim.x) {
    const uint32_t sy = static_cast<uint32_t>(key[i]) ^ 0x80000000u;
    hv.syms[i] = static_cast<int32_t>(sy);
    if (ssym) ssym[i] = sy;
  }
  if (threadIdx.x < 33) {
    tb.count[threadIdx.x] = 0;
    tb.first[threadIdx.x] = 0;
    tb.base[threadIdx.x] = 0;
  }
  __syncthreads();
  // canonical codes (closed form of finalize's shift-and-increment)
  const double w = 2.0 * S.eb;
  unsigned long long carry = 0;
  for (uint32_t i0 = 0; i0 < nent; i0 += blockDim.x) {
    const uint32_t i = i0 + threadIdx.x;
    uint32_t len = 0;
    unsigned long long k = 0;
    if (i < nent) {
      len = static_cast<uint32_t>(key[i] >> 32);
      k = 1ull << (32 - len);
    }
    unsigned long long tot;
    const unsigned long long pre = block_excl_scan<unsigned long long>(k, s_tmp64, &tot);
    if (i < nent) {
      const uint32_t code = static_cast<uint32_t>((carry + pre) >> (32 - len));
      const bool first_of_len = (i == 0) || static_cast<uint32_t>(key[i - 1] >> 32) != len;
      if (first_of_len) {
        tb.first[len] = code;
        tb.base[len] = i;
      }
      atomicAdd(&tb.count[len], 1u);
      hv.vals[i] = value_bits(static_cast<int32_t>(static_cast<uint32_t>(key[i]) ^ 0x80000000u), w, C.out_kind);
    }
    carry += tot;
  }
  __syncthreads();
  DTS(8000 + c, 4);
  // left-aligned code starts, ascending in canonical order -> prefix LUT
  for (uint32_t i = threadIdx.x; i < nent; i += blockDim.x) {
    const uint32_t len = static_cast<uint32_t>(key[i] >> 32);
    // code_i = first[len] + (i - base[len])
    const uint64_t code = tb.first[len] + (i - tb.base[len]);
    key[i] = (code << (32 - len)) | (static_cast<uint64_t>(len) << 56);  // start < 2^32; len in top byte
  }
  __syncthreads();
  for (uint32_t s = threadIdx.x; s < (1u << kL0); s += blockDim.x) {
    const uint64_t V = static_cast<uint64_t>(s) << (32 - kL0);
    const uint64_t Vend = V + (1ull << (32 - kL0));
    // last entry with start <= V
    int lo = 0, hi = static_cast<int>(nent) - 1, f = -1;
    while (lo <= hi) {
      const int mid = (lo + hi) >> 1;
      if ((key[mid] & 0xFFFFFFFFFFull) <= V) {
        f = mid;
        lo = mid + 1;
      } else {
        hi = mid - 1;
      }
    }
    uint32_t ent = 0;
    if (f >= 0) {
      const uint32_t len = static_cast<uint32_t>(key[f] >> 56);
      const uint64_t a = key[f] & 0xFFFFFFFFFFull;
      if (V < a + (1ull << (32 - len))) ent = len <= kL0 ? (static_cast<uint32_t>(f) << 6) | len : kLong;
    }
    if (!ent && f + 1 < static_cast<int>(nent) && (key[f + 1] & 0xFFFFFFFFFFull) < Vend) ent = kLong;
    hv.lut[s] = ent;
  }
  __syncthreads();  // the code starts in key[] are read above; reused below
  DTS(8000 + c, 5);
  // duplicate symbols (huffman.hpp:183-185) across all lengths
  for (uint32_t i = threadIdx.x; i < p2; i += blockDim.x)
    key[i] = i < nent ? (static_cast<uint64_t>((ssym ? ssym[i] : static_cast<uint32_t>(hv.syms[i])) ^ 0x80000000u) << 32) | i
                      : ~0ull;
  __syncthreads();
  if (ssym && p2 <= 256) {
    if (threadIdx.x < 32) warp_sort_smem(key, p2);
    __syncthreads();
  } else {
    bitonic_sort_u64(key, p2);
  }
  DTS(8000 + c, 6);
  bool dup = false;
  for (uint32_t i = 1 + threadIdx.x; i < nent; i += blockDim.x) dup |= (key[i] >> 32) == (key[i - 1] >> 32);
  dup = __syncthreads_or(dup);
  if (dup) {
    if (threadIdx.x == 0) dec_fail(S, 0, EMBC_R_HUF_DUP, 0, 0);
    return;
  }
  if (threadIdx.x == 0) {
    uint32_t max_len = 0;  // entries().back().length (huffman.hpp:257)
    for (uint32_t l = 1; l <= 32; ++l)
      if (tb.count[l]) max_len = l;
    tb.max_len = max_len;
    tb.nent = nent;
    tb.nsym = S.nsym;
    tb.bit_off = 12 + 5ull * nent;
    tb.nbits = 8 * (L - tb.bit_off);
    *hv.tab = tb;
    S.max_len = max_len;
    S.bit_off = tb.bit_off;
    if (S.nsym != C.N) hflag[c] = 1;  // decoded count != dim*count (container.hpp:169-172)
  }
}

// 32 bits starting at bit `pos` of the stream (zeros past the end).
__device__ __forceinline__ uint32_t peek32(const uint8_t* s, uint64_t nbytes, uint64_t pos) {
  const uint64_t byte = pos >> 3;
  const uint32_t sh = static_cast<uint32_t>(pos & 7);
  uint64_t w = 0;
  if (byte + 5 <= nbytes) {
#pragma unroll
    for (int k = 0; k < 5; ++k) w = (w << 8) | s[byte + k];
  } else {
    for (int k = 0; k < 5; ++k) w = (w << 8) | (byte + k < nbytes ? s[byte + k] : 0);
  }
  return static_cast<uint32_t>(w >> (8 - sh));
}

// One canonical codeword at `pos`: returns entry index and sets *len, or -1
// if no codeword matches (invalid prefix).
__device__ __forceinline__ int decode_one(const uint32_t* lut, const HTab& t, uint32_t bits, uint32_t* len) {
  const uint32_t e = lut[bits >> (32 - kL0)];
  if (e != kLong) {
    if (!e) return -1;
    *len = e & 63;
    return static_cast<int>(e >> 6);
  }
  for (uint32_t l = kL0 + 1; l <= t.max_len; ++l) {
    const uint32_t code = bits >> (32 - l);
    if (t.count[l] && code >= t.first[l] && code - t.first[l] < t.count[l]) {
      *len = l;
      return static_cast<int>(t.base[l] + (code - t.first[l]));
    }
  }
  return -1;
}

// Packed map entry: entry/exit bit offset (5 bits) | termination kind (2 bits)
// | symbol count (25 bits).  Termination: 0 live, 1 invalid prefix, 2 stream end.
__device__ __forceinline__ uint32_t pk(uint32_t off, uint32_t term, uint32_t cnt) {
  return off | (term << 5) | (cnt << 7);
}
__device__ __forceinline__ uint32_t pk_off(uint32_t v) { return v & 31; }
__device__ __forceinline__ uint32_t pk_term(uint32_t v) { return (v >> 5) & 3; }
__device__ __forceinline__ uint32_t pk_cnt(uint32_t v) { return v >> 7; }

// Stage the CTA's slice of the bitstream as big-endian 32-bit words.
__device__ __forceinline__ void stage_bits(uint32_t* W, uint32_t nwords, const uint8_t* s, uint64_t nbytes, uint64_t bit0) {
  const uint64_t b0 = bit0 >> 3;  // bit0 is a multiple of 32
  for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x) {
    const uint64_t b = b0 + 4ull * w;
    uint32_t v = 0;
    if (b + 4 <= nbytes) {
      v = (static_cast<uint32_t>(s[b]) << 24) | (static_cast<uint32_t>(s[b + 1]) << 16) |
          (static_cast<uint32_t>(s[b + 2]) << 8) | s[b + 3];
    } else {
      for (int k = 0; k < 4; ++k) v = (v << 8) | (b + k < nbytes ? s[b + k] : 0);
    }
    W[w] = v;
  }
}

// The five staged words around one subsequence (two before it, its two, one
// after) in registers: 32 bits at bit offset pos in [-64, 64) of the
// subsequence without a shared-memory access on the decode chain.
struct SubWin {
  uint32_t a0, a1, a2, a3, a4;
  __device__ __forceinline__ SubWin(const uint32_t* W, uint32_t w0)
      : a0(W[w0 - 2]), a1(W[w0 - 1]), a2(W[w0]), a3(W[w0 + 1]), a4(W[w0 + 2]) {}
  __device__ __forceinline__ uint32_t peek(int pos) const {
    const uint32_t k = static_cast<uint32_t>(pos + 64) >> 5;  // 0..3
    const uint32_t hi = k == 0 ? a0 : k == 1 ? a1 : k == 2 ? a2 : a3;
    const uint32_t lo = k == 0 ? a1 : k == 1 ? a2 : k == 2 ? a3 : a4;
    return __funnelshift_l(lo, hi, static_cast<uint32_t>(pos) & 31);
  }
};

// 32 bits at relative bit position p of the staged words.
__device__ __forceinline__ uint32_t speek(const uint32_t* W, uint32_t p) {
  const uint32_t i = p >> 5;
  return __funnelshift_l(W[i + 1], W[i], p & 31);
}

__device__ __forceinline__ uint32_t popc_below(uint64_t bm, uint32_t p) {
  return static_cast<uint32_t>(__popcll(bm & ((1ull << p) - 1ull)));
}
// Exact sequential walk (huffman.hpp:274-290) for flagged chunks: reproduces
// the reference's first error (exhaustion / invalid prefix / count).
EMBC_COLD void k_dec_huff_seq_cta(uint32_t bid, const DChunk* __restrict__ ch, DecState* __restrict__ st,
                               const uint32_t* list, uint8_t* tabs, const volatile uint32_t* hflag) {
  if (threadIdx.x != 0) return;
  const uint32_t c = bid;
  const DChunk C = ch[c];
  DecState& S = st[c];
  if (S.err != ~0ull || !hflag[c]) return;
  HView hv = hview(tabs, C);
  const HTab& tb = *hv.tab;
  const uint8_t* bits = C.in + S.pay_off + tb.bit_off;
  const uint64_t nbytes = tb.nbits / 8;
  const uint64_t nsym = tb.nsym;
  uint64_t byte = 0;
  uint32_t shift = 0;
  for (uint64_t i = 0; i < nsym; ++i) {
    uint32_t code = 0, len = 0;
    for (;;) {
      if (byte >= nbytes) {
        dec_fail(S, i, EMBC_R_HUF_EXHAUSTED, 8 * byte, 0);
        return;
      }
      const uint32_t b = (bits[byte] >> (7 - shift)) & 1u;
      if (++shift == 8) {
        shift = 0;
        ++byte;
      }
      code = (code << 1) | b;
      ++len;
      if (tb.count[len] != 0 && code >= tb.first[len] && code - tb.first[len] < tb.count[len]) {
        if (i < C.N) {
          const uint64_t v = hv.vals[tb.base[len] + (code - tb.first[len])];
          if (C.out_kind == EMBC_OUT_F64) static_cast<uint64_t*>(C.out)[i] = v;
          else static_cast<uint32_t*>(C.out)[i] = static_cast<uint32_t>(v);
        }
        break;
      }
      if (len >= tb.max_len) {
        dec_fail(S, i, EMBC_R_HUF_BAD_CODE, 0, 0);
        return;
      }
    }
  }
  if (nsym != C.N) dec_fail(S, 0, EMBC_R_HUF_COUNT, nsym, C.N);
}

// ---------------------------------------------------------------------------
// D9: fold the lowest failing chunk into the sticky record.
// ---------------------------------------------------------------------------
// The lowest failing chunk -> the sticky record (all threads of the CTA scan).
EMBC_COLD void dec_fold(const DecState* __restrict__ st, uint32_t n, DevError* err) {
  __shared__ uint32_t s_first;
  if (threadIdx.x == 0) s_first = 0xFFFFFFFFu;
  __syncthreads();
  for (uint32_t c = threadIdx.x; c < n; c += blockDim.x)
    if (__ldcg(reinterpret_cast<const unsigned long long*>(&st[c].err)) != ~0ull) atomicMin(&s_first, c);
  __syncthreads();
  if (threadIdx.x != 0 || s_first == 0xFFFFFFFFu || err->valid) return;
  const uint32_t c = s_first;
  const DecState& S = st[c];
  err->valid = 1;
  err->job = c;
  err->reason = static_cast<int32_t>(S.err & 63);
  err->index = S.err >> 6;
  err->a = S.a;
  err->b = S.b;
  err->eb = S.eb;
  const int r = err->reason;
  err->status = (r == EMBC_R_BAD_EB) ? EMBC_ERR_VALUE : (r == EMBC_R_RANGE) ? EMBC_ERR_UNSUPPORTED : EMBC_ERR_FORMAT;
}

// ===========================================================================
// look-back status words (flag in bits 63:62; 1 = aggregate map published,
// 2 = inclusive state published)
// ===========================================================================
constexpr unsigned long long kStAgg = 1ull << 62, kStInc = 2ull << 62;

__device__ __forceinline__ unsigned long long ld_vol(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}
// Status store without a fence: for an aggregate flag whose data every writer
// fenced before a barrier the storing thread passed, and for inclusive states
// (values that publish no other data).
__device__ __forceinline__ void st_flag(unsigned long long* p, unsigned long long v) {
  *reinterpret_cast<volatile unsigned long long*>(p) = v;
}
__device__ __forceinline__ void st_vol(unsigned long long* p, unsigned long long v) {
  __threadfence();
  *reinterpret_cast<volatile unsigned long long*>(p) = v;
}

// Warp 0: index of the nearest predecessor in [first, i) with an inclusive
// state (every element between it and i has at least published its map).
// Returns that index and its status word.
__device__ __forceinline__ uint32_t find_inclusive(const unsigned long long* status, uint32_t first, uint32_t i,
                                                   unsigned long long* word) {
  const uint32_t lane = threadIdx.x & 31;
  int64_t p = static_cast<int64_t>(i) - 1;
  uint32_t delay = 32;
  for (;;) {
    const int64_t idx = p - lane;
    unsigned long long s = kStInc;
    if (idx >= static_cast<int64_t>(first)) s = ld_vol(status + idx);
    const uint32_t inc = __ballot_sync(0xffffffffu, (s >> 62) == 2);
    const uint32_t zero = __ballot_sync(0xffffffffu, (s >> 62) == 0);
    const int fi = inc ? __ffs(inc) - 1 : 32;
    const uint32_t need = fi == 32 ? 0xffffffffu : ((2u << fi) - 1);
    if (zero & need) {  // a predecessor has not published yet: back off, re-read
      __nanosleep(delay);
      delay = min(delay * 2, kPollMaxNs);
      continue;
    }
    if (fi < 32) {
      *word = __shfl_sync(0xffffffffu, s, fi);
      return static_cast<uint32_t>(p - fi);
    }
    p -= 32;
  }
}

// ===========================================================================
// VLZ (vlz.hpp:129-158) without its sequential dependency.
//
// A valid token stream is a sequence of "units": maximal byte runs ending in a
// byte with bit 7 clear.  Tags are one-byte units (0x00 / 0x01) and every
// varint is one unit, so the token chain over units is
// next(u) = u + (tag 0x00 ? dim + 1 : 2).  Each 2 KiB segment builds binary
// lifting tables of that chain, derives its entry -> (exit, tokens) map for
// the dim + 1 possible entry offsets, and learns its true entry from the
// segments before it (decoupled look-back).  Any anomaly flags the chunk;
// the exact sequential walker then reproduces the reference's error.
// ===========================================================================
constexpr uint32_t kSeg = 1024;         // payload bytes per segment
constexpr uint32_t kVlzMaxDim = 1023;   // larger dims use the sequential walker
constexpr int kLift = 10;               // 2^10 > kSeg / 2 tokens per segment
constexpr uint16_t kInv = 0xFFFF;
constexpr uint32_t kSegBack = 16;       // bytes staged before the segment (first unit's start)
// VLZ segment smem for chunks of dim <= dmax: staged bytes (the segment plus
// one literal token past it) | unit ends | lifting tables | literal queue
__host__ __device__ constexpr uint32_t vlz_unit_cap(uint32_t dmax) { return kSeg + dmax + 2; }
__host__ __device__ constexpr uint32_t vlz_bytes_cap(uint32_t dmax) {
  return (kSegBack + kSeg + 10 * (dmax + 1) + 32 + 15) & ~15u;
}
__host__ __device__ constexpr uint32_t vlz_smem(uint32_t dmax) {
  return vlz_bytes_cap(dmax) + ((vlz_unit_cap(dmax) * 2 + 15) & ~15u) + kLift * kSeg * 2 + 8 * (kSeg / 2);
}
constexpr uint32_t kVlzSmem = vlz_smem(kVlzMaxDim);

// huffman block descriptor: staging the block needs no chunk descriptor
struct HBlkDesc {
  uint32_t chunk, blk;
  const uint8_t* in;
  uint64_t length;
};

// vlz segment descriptor: the chunk, the segment, and what staging the
// segment's bytes needs, so the bytes load right after this descriptor (the
// chunk descriptor and the header check follow off the critical path)
struct SegPair {
  uint32_t chunk, seg;
  const uint8_t* in;  // the chunk's first byte
  uint32_t length;    // the chunk's bytes (< 2^31 for a parallel-decoded chunk)
  uint32_t dim;
};

// inclusive vlz state: flag | dead (61) | entry unit offset (42:32) | rows (31:0)
__device__ __forceinline__ unsigned long long vlz_state(bool dead, uint32_t e, uint32_t rows) {
  return (dead ? (1ull << 61) : 0) | (static_cast<unsigned long long>(e & 0x7FF) << 32) | rows;
}

struct DecArgs {
  const DChunk* ch;
  DecState* st;
  const SegPair* segs;
  const uint32_t* hblk_chunk;  // huffman block -> chunk
  const struct HBlkDesc* hblk; // huffman block -> (chunk, block in chunk, chunk bytes)
  const RawTile* raw;
  const uint32_t* ctile;       // D2 copy tiles: (chunk << 0) in [0], row0 in [1], rows in [2] (triplets)
  uint32_t* vflag;
  uint32_t* hflag;
  uint32_t* ready;
  uint32_t* cnt;               // per-chunk tail tickets
  uint32_t* vdone;             // per chunk: vlz segments finished (the last one after the roots)
  uint32_t* hdone;             // per chunk: huffman blocks finished
  uint32_t* tickets;           // [0] role ticket, [1] fold ticket, [2] fallback count
  unsigned long long* seg_status;
  unsigned long long* blk_status;
  uint32_t* maps;              // vlz: per segment (dim + 1) entry maps
  uint32_t* bmaps;             // huffman: per block 32 entry maps
  uint32_t* row_src;
  uint64_t* keys;
  uint8_t* tabs;
  DevError* err;
  uint32_t* diag;
  uint32_t nchunks, nseg, nhblk, nraw, nctile;
  uint32_t vlz_dmax;    // largest vlz dim of the call (sizes the segment smem carve)
  uint32_t hsub;        // subsequences per huffman block
  uint32_t sbits;       // bits per subsequence (32 or 64)
  uint32_t local_tables;  // small calls: every huffman block builds its own decode tables
  uint32_t smem_bytes;  // dynamic shared memory of k_dec_main
  const uint32_t* dcount;  // device-planned calls: [0] vlz segments, [1] huffman blocks (else null)
  uint32_t persistent;     // CTAs loop over role tickets (device-planned calls)
  uint32_t payload_only;   // chunks are bare payloads (no header)
};

__device__ __forceinline__ uint64_t stage_varint(const uint8_t* B, uint32_t start, uint32_t end) {
  uint64_t v = 0;
  int shift = 0;
  for (uint32_t k = start; k <= end; ++k, shift += 7)
    if (shift < 64) v |= static_cast<uint64_t>(B[k] & 0x7F) << shift;
  return v;
}

__device__ void vlz_end_check(const DecArgs& a, uint32_t c);
__device__ __forceinline__ bool vlz_roots_local(const DecArgs& a, const DChunk& C);
__device__ void vlz_resolve_roots(const DecArgs& a, const DChunk& C, uint8_t* smem);

EMBC_ROLE void vlz_segment(const DecArgs& a, uint32_t gseg, uint8_t* smem) {
  __shared__ uint32_t s_tmp32[33];
  __shared__ uint32_t s_bad, s_nlit, s_first_start;
  __shared__ unsigned long long s_in;
  __shared__ int s_last;
  const SegPair sp = a.segs[gseg];
  const uint32_t c = sp.chunk;
  // the chunk descriptor, copied to shared memory by the last warp while the
  // other threads stage the segment's bytes (read after the unit-table barriers)
  __shared__ __align__(8) DChunk sC;
  const DChunk& C = sC;
  __shared__ unsigned long long s_err;
  __shared__ double s_eb;
  DROLE(blockIdx.x, 1);
  const uint32_t D = sp.dim;
  __shared__ uint8_t s_hdr[32];
  if (threadIdx.x >= blockDim.x - 32) {  // with the header bytes, in the same round
    const uint32_t l = threadIdx.x - (blockDim.x - 32);
    if (l < sizeof(DChunk) / 8)
      reinterpret_cast<unsigned long long*>(&sC)[l] = __ldg(reinterpret_cast<const unsigned long long*>(a.ch + c) + l);
    s_hdr[l] = (!a.payload_only && l < kHeader && l < sp.length) ? __ldg(sp.in + l) : 0;
  }
  const uint32_t kUnitCap = vlz_unit_cap(a.vlz_dmax);
  uint8_t* B = smem;                                                          // staged bytes (set below)
  uint16_t* uend = reinterpret_cast<uint16_t*>(smem + vlz_bytes_cap(a.vlz_dmax));  // unit terminal byte
  uint16_t(*J)[kSeg] = reinterpret_cast<uint16_t(*)[kSeg]>(reinterpret_cast<uint8_t*>(uend) + ((kUnitCap * 2 + 15) & ~15u));
  uint32_t* lit = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(J) + kLift * kSeg * 2);  // literal tokens (<= kSeg/2)
  // the payload's place follows from the plan (the host cut the segments from
  // length - header); the header is validated by thread 0 while the bytes load
  const uint64_t poff = a.payload_only ? 0 : kHeader;
  const uint8_t* p = sp.in + poff;
  const uint64_t L = sp.length - poff;
  const uint32_t b0 = sp.seg * kSeg;
  const uint32_t nb = static_cast<uint32_t>(umin64(kSeg, L - b0));
  const uint32_t sb = b0 >= kSegBack ? b0 - kSegBack : 0;
  const uint32_t la = static_cast<uint32_t>(umin64(L - (b0 + nb), 10ull * (D + 1) + 10));
  const uint32_t ns = b0 + nb + la - sb;
  {  // 16-B loads of the aligned blocks covering [sb, sb + ns); B points at byte sb
    const uintptr_t g0 = reinterpret_cast<uintptr_t>(p + sb);
    const uint4* gv = reinterpret_cast<const uint4*>(g0 & ~uintptr_t(15));
    const uint32_t lead = static_cast<uint32_t>(g0 & 15);
    const uint32_t nv = (lead + ns + 15) / 16;
    uint4* sv = reinterpret_cast<uint4*>(smem);
    for (uint32_t k0 = 0; k0 < nv; k0 += 4 * blockDim.x) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t k = k0 + u * blockDim.x + threadIdx.x;
        if (k < nv) v[u] = __ldg(gv + k);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t k = k0 + u * blockDim.x + threadIdx.x;
        if (k < nv) sv[k] = v[u];
      }
    }
    B = smem + lead;
  }
  if (threadIdx.x == 0) {
    s_bad = 0;
    s_nlit = 0;
  }
  __syncthreads();
  // header check (parse_chunk on the staged header bytes); its verdict is
  // read before the segment publishes anything
  if (threadIdx.x == 0) {
    const DecState S = parse_chunk_hb(C, s_hdr);
    s_err = S.err;
    s_eb = S.eb;
  }
  DTS(blockIdx.x, 2);
  // unit table: terminal bytes at payload offsets [b0, b0 + nb + la)
  uint32_t nu = 0, U = 0;
  for (uint32_t r0 = b0; r0 < b0 + nb + la && nu < kUnitCap; r0 += 8 * blockDim.x) {
    const uint32_t x0 = r0 + threadIdx.x * 8;
    uint32_t mask = 0, nseg_here = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (x0 + k < b0 + nb + la && !(B[x0 + k - sb] & 0x80)) {
        mask |= 1u << k;
        nseg_here += x0 + k < b0 + nb;
      }
    // one scan for both counts: units of the round (low half) and units ending
    // inside the segment (high half; the segment lies in the first round)
    uint32_t tot;
    const uint32_t ex = block_excl_scan<uint32_t>(__popc(mask) | (nseg_here << 16), s_tmp32, &tot);
    uint32_t k0 = nu + (ex & 0xFFFF);
    if (r0 == b0) U = tot >> 16;
    tot &= 0xFFFF;
    uint32_t m = mask;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      if (k0 < kUnitCap) uend[k0] = static_cast<uint16_t>(x0 + b - sb);
      ++k0;
    }
    nu += tot;
  }
  nu = min(nu, kUnitCap);
  if (threadIdx.x == 0) {  // the first unit may begin in the previous segment
    uint32_t start = b0;  // walks back at most 11 bytes, inside the kSegBack staged before the segment
    while (start > 0 && (B[start - 1 - sb] & 0x80) && b0 - start <= 10) --start;
    s_first_start = start - sb;
    // a trailing partial unit can never be consumed by a valid parse
    if (b0 + nb == L && nb > 0 && (B[L - 1 - sb] & 0x80)) s_bad = 1;
  }
  __syncthreads();
  DTS(blockIdx.x, 3);
  auto ustart = [&](uint32_t k) -> uint32_t { return k ? uend[k - 1] + 1u : s_first_start; };
  // unit kinds -> level-0 jumps; units longer than 10 bytes are never valid (bytes.hpp:139-147)
  for (uint32_t k = threadIdx.x; k < U; k += blockDim.x) {
    const uint32_t st0 = ustart(k), e = uend[k];
    const uint32_t len = e - st0 + 1;
    if (len > 10) s_bad = 1;
    const uint8_t v = B[st0];
    const uint32_t kind = (len == 1 && v <= 1) ? v : 2;
    J[0][k] = kind == 2 ? kInv : static_cast<uint16_t>(k + (kind == 0 ? D + 1 : 2));
  }
  __syncthreads();
  int nlev = kLift;  // levels past the point where every jump has left the segment are copies
  for (int r = 1; r < kLift; ++r) {
    bool live = false;
    for (uint32_t k0 = threadIdx.x; k0 < U; k0 += 4 * blockDim.x) {  // four units in flight
      uint16_t j[4], v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t k = k0 + u * blockDim.x;
        j[u] = k < U ? J[r - 1][k] : kInv;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = (j[u] == kInv || j[u] >= U) ? j[u] : J[r - 1][j[u]];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t k = k0 + u * blockDim.x;
        if (k < U) {
          J[r][k] = v[u];
          live |= v[u] != kInv && v[u] < U;
        }
      }
    }
    if (!__syncthreads_or(live)) {
      nlev = r + 1;
      break;
    }
  }
  DTS(blockIdx.x, 4);
  if (s_err != ~0ull) return;  // every CTA of the chunk sees it: nobody waits on this segment
  // entry -> (exit offset into the next segment, tokens) for entries 0..D
  uint32_t* mymap = a.maps + C.map_base + static_cast<uint64_t>(sp.seg) * (D + 1);
  for (uint32_t e = threadIdx.x; e <= D; e += blockDim.x) {
    uint32_t m;
    if (e >= U) {
      m = e - U;  // no token starts in this segment
    } else {
      uint32_t pos = e, n = 0;
      for (int r = nlev - 1; r >= 0; --r) {
        const uint16_t j = J[r][pos];
        if (j != kInv && j < U) {
          pos = j;
          n += 1u << r;
        }
      }
      const uint16_t x = J[0][pos];
      m = x == kInv ? 0xFFFFFFFFu : (((n + 1) << 16) | (x - U));
    }
    mymap[e] = m;
  }
  __threadfence();
  __syncthreads();
  DTS(blockIdx.x, 5);
  unsigned long long* status = a.seg_status;
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0 && sp.seg > 0) st_flag(status + gseg, kStAgg);  // maps fenced before the barrier
    unsigned long long in;
    if (sp.seg == 0) {
      in = vlz_state(false, 0, 0);
    } else {
      unsigned long long w;
      const uint32_t q = find_inclusive(status, C.seg0, gseg, &w);
      bool dead = (w >> 61) & 1;
      uint32_t e = static_cast<uint32_t>(w >> 32) & 0x7FF, rows = static_cast<uint32_t>(w);
      // apply the maps published after it: batches loaded in parallel into
      // shared memory (the literal queue is free until the tokens), applied in order
      const uint32_t cap = max(1u, kSeg / (D + 1));  // lit holds kSeg u32
      for (uint32_t m0 = q + 1; m0 < gseg && !dead; m0 += cap) {
        const uint32_t nm = min(cap, gseg - m0);
        const uint32_t* src = a.maps + C.map_base + static_cast<uint64_t>(m0 - C.seg0) * (D + 1);
        for (uint32_t k = threadIdx.x; k < nm * (D + 1); k += 32) lit[k] = __ldcg(src + k);
        __syncwarp();
        for (uint32_t m = 0; m < nm && !dead; ++m) {
          const uint32_t v = lit[m * (D + 1) + e];
          if (v == 0xFFFFFFFFu) dead = true;
          else {
            rows += v >> 16;
            e = v & 0xFFFF;
          }
        }
        __syncwarp();
      }
      in = vlz_state(dead, e, rows);
    }
    if (threadIdx.x == 0) {
      bool dead = (in >> 61) & 1;
      const uint32_t e = static_cast<uint32_t>(in >> 32) & 0x7FF, rows = static_cast<uint32_t>(in);
      uint32_t eo = 0, ro = rows;
      if (!dead) {
        const uint32_t v = mymap[e];
        if (v == 0xFFFFFFFFu) dead = true;
        else {
          eo = v & 0xFFFF;
          ro = rows + (v >> 16);
          if (ro > C.count) dead = true;  // more tokens than vectors: trailing bytes
        }
      }
      st_flag(status + gseg, kStInc | vlz_state(dead, eo, ro));
      s_in = in;
    }
  }
  __syncthreads();
  DTS(blockIdx.x, 6);
  const unsigned long long in = s_in;
  const bool dead_in = (in >> 61) & 1;
  const uint32_t e_in = static_cast<uint32_t>(in >> 32) & 0x7FF, row0 = static_cast<uint32_t>(in);
  bool bad = s_bad || dead_in;
  const uint32_t T = (!bad && e_in < U) ? (mymap[e_in] == 0xFFFFFFFFu ? 0 : mymap[e_in] >> 16) : 0;
  if (!bad && e_in < U && mymap[e_in] == 0xFFFFFFFFu) bad = true;
  if (!bad && row0 + T > C.count) bad = true;
  // every token of the segment: reference offsets validated (vlz.hpp:141-145),
  // literal tokens queued for the warp decoder
  const double w = 2.0 * s_eb;
  uint32_t* row_src = a.row_src + C.row_base;
  if (!bad) {
    for (uint32_t t = threadIdx.x; t < T; t += blockDim.x) {
      uint32_t u = e_in;
      for (int r = 0; r < nlev; ++r)
        if ((t >> r) & 1) u = J[r][u];
      const uint32_t row = row0 + t;
      const uint8_t tag = B[uend[u]];
      if (tag == 0x01) {
        if (u + 1 >= nu) {
          s_bad = 1;
          continue;
        }
        const uint32_t s1 = ustart(u + 1), e1 = uend[u + 1];
        if (e1 - s1 + 1 > 10) {
          s_bad = 1;
          continue;
        }
        const uint64_t off = stage_varint(B, s1, e1);
        if (off < 1 || off > row || off > kMaxWindow) {
          s_bad = 1;
          continue;
        }
        row_src[row] = row - static_cast<uint32_t>(off);
      } else {
        row_src[row] = row;
        const uint32_t k = atomicAdd(&s_nlit, 1u);
        lit[2 * k] = row;
        lit[2 * k + 1] = u;
      }
    }
  }
  __syncthreads();
  DTS(blockIdx.x, 8);
  if (!bad) {  // literal rows: 0x00 then dim zigzag varints, one warp per row
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t nl = s_nlit;
    for (uint32_t q = warp; q < nl; q += nw) {
      const uint32_t row = lit[2 * q], u = lit[2 * q + 1];
      for (uint32_t j = lane; j < D; j += 32) {
        const uint32_t k = u + 1 + j;
        if (k >= nu) {
          s_bad = 1;
          break;
        }
        const uint32_t s1 = ustart(k), e1 = uend[k];
        if (e1 - s1 + 1 > 10) {
          s_bad = 1;
          break;
        }
        store_value(C, static_cast<uint64_t>(row) * D + j, unzigzag(static_cast<uint32_t>(stage_varint(B, s1, e1))), w);
      }
    }
  }
  __syncthreads();
  DTS(blockIdx.x, 9);
  if (threadIdx.x == 0 && (bad || s_bad)) atomicOr(&a.vflag[c], 1u);
  // the chunk's last segment to finish checks the end state
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&a.cnt[c], 1u) == C.nseg - 1;
  __syncthreads();
  DTS(blockIdx.x, 10);
  if (!s_last) return;
  __threadfence();
  vlz_end_check(a, c);
  __syncthreads();
  if (vlz_roots_local(a, C) && !*reinterpret_cast<volatile uint32_t*>(&a.vflag[c])) {
    vlz_resolve_roots(a, C, smem);
  }
  DTS(blockIdx.x, 11);
}

// Reference rows are copied from their roots (the first occurrence of the
// row: row_src == itself); a row's source is always an earlier row.  When the
// chunk's row sources fit in shared memory, its last segment resolves every
// row's root there once (pointer jumping, four rows in flight per thread) and
// writes the roots back, so the copy tiles only copy.  Larger chunks leave the
// jumping to the copy tiles (through L2).
__device__ __forceinline__ bool vlz_roots_local(const DecArgs& a, const DChunk& C) {
  return static_cast<uint64_t>(C.count) * 4 <= a.smem_bytes;
}

__device__ void vlz_resolve_roots(const DecArgs& a, const DChunk& C, uint8_t* smem) {
  uint32_t* V = reinterpret_cast<uint32_t*>(smem);
  uint32_t* src = a.row_src + C.row_base;
  const uint32_t n = C.count;
  for (uint32_t q0 = 0; q0 < n; q0 += 4 * blockDim.x) {
    uint32_t v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t r = q0 + u * blockDim.x + threadIdx.x;
      v[u] = r < n ? __ldcg(src + r) : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t r = q0 + u * blockDim.x + threadIdx.x;
      if (r < n) V[r] = v[u];
    }
  }
  __syncthreads();
  for (;;) {
    bool changed = false;
    for (uint32_t q0 = 0; q0 < n; q0 += 4 * blockDim.x) {
      uint32_t v[4], w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t r = q0 + u * blockDim.x + threadIdx.x;
        v[u] = r < n ? V[r] : 0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = V[v[u]];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t r = q0 + u * blockDim.x + threadIdx.x;
        if (r < n && w[u] != v[u]) {
          V[r] = w[u];
          changed = true;
        }
      }
    }
    if (!__syncthreads_or(changed)) break;
  }
  for (uint32_t r = threadIdx.x; r < n; r += blockDim.x) __stcg(src + r, V[r]);
}

// The chunk's end state after its last segment (vlz.hpp:154-157): the token
// chain must end exactly at the payload end with one vector per row.
__device__ void vlz_end_check(const DecArgs& a, uint32_t c) {
  if (threadIdx.x != 0) return;
  const DChunk& C = a.ch[c];
  const unsigned long long w = ld_vol(a.seg_status + C.seg0 + C.nseg - 1);
  const bool dead = (w >> 61) & 1;
  const uint32_t e = static_cast<uint32_t>(w >> 32) & 0x7FF, rows = static_cast<uint32_t>(w);
  if (dead || rows != C.count || e != 0) a.vflag[c] = 1;
}

// ===========================================================================
// Huffman blocks: 128 subsequences of 64 bits.
// ===========================================================================
constexpr uint32_t kHSub = 256;                        // subsequences per block (one per thread)
constexpr uint32_t kMaxGroups = 32;                    // group walks per block (8 warps, up to four each)
constexpr uint32_t kHPre = 2;                          // words staged before the block (warm-up)
// smem: LUT | two-codeword LUT | staged words | per-subsequence chain summaries | group states, later the symbols (u16)
__host__ __device__ constexpr uint32_t huff_smem(uint32_t hsub, uint32_t sbits = kSubBits) {
  return (1u << kL0) * 4 + (1u << kL0) * 2 + (((kHPre + hsub * sbits / 32 + 4) * 4 + 15) & ~15u) + hsub * 20 +
         (hsub * 33 * 4 > hsub * sbits * 2 ? hsub * 33 * 4 : hsub * sbits * 2);
}
constexpr uint32_t kHuffSmem = huff_smem(kHSub);

// inclusive huffman state: flag | term (61:60) | entry bit offset (59:55) | symbols (54:0)
__device__ __forceinline__ unsigned long long huf_state(uint32_t term, uint32_t e, uint64_t cnt) {
  return (static_cast<unsigned long long>(term & 3) << 60) | (static_cast<unsigned long long>(e & 31) << 55) |
         (cnt & ((1ull << 55) - 1));
}

// Huffman block (16384 bits = 256 subsequences of 64 bits, one per thread):
//  A  every subsequence decodes one chain that starts 64 bits early (in the
//     previous subsequence), so it has usually synchronised with the true
//     codeword boundaries by the time it enters: its starts inside the
//     subsequence (bitmap), exit and symbol count.  A second chain starts at
//     the previous subsequence's exit and runs until it lands on one of those
//     starts.
//  B  per group of 32 subsequences, lane r follows entry offset r: a known
//     start or the precomputed entry resolves in O(1), anything else decodes
//     until it lands on a start.  Group and block maps then give the block's
//     entry -> (exit, symbols) map, published for a decoupled look-back over
//     the chunk's earlier blocks.
//  C  with the true entry known, every subsequence decodes its symbols into
//     shared memory; the block stores them coalesced.
EMBC_ROLE void huff_block(const DecArgs& a, uint32_t gb, uint8_t* smem) {
  __shared__ HTab t;
  __shared__ uint32_t G[kMaxGroups][32], BM[32];
  __shared__ unsigned long long s_in;
  __shared__ int s_use;
  const HBlkDesc hd = a.hblk[gb];
  const uint32_t c = hd.chunk;
  // the chunk descriptor, copied to shared memory by the last warp while the
  // chunk's first bytes load (read after the barrier below)
  __shared__ __align__(8) DChunk sC;
  const DChunk& C = sC;
  if (threadIdx.x >= blockDim.x - 32) {
    const uint32_t l = threadIdx.x - (blockDim.x - 32);
    if (l < sizeof(DChunk) / 8)
      reinterpret_cast<unsigned long long*>(&sC)[l] = __ldg(reinterpret_cast<const unsigned long long*>(a.ch + c) + l);
  }
  const uint32_t b = hd.blk;
  const uint32_t hsub = a.hsub, SB = a.sbits, SW = SB / 32, hbits = hsub * SB, hwords = kHPre + hbits / 32 + 4;
  uint32_t* lut = reinterpret_cast<uint32_t*>(smem);
  uint16_t* luta = reinterpret_cast<uint16_t*>(lut + (1u << kL0));  // two-codeword steps (lengths only)
  uint32_t* W = lut + (1u << kL0) + (1u << kL0) / 2;
  uint64_t* B0 = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(W) + ((hwords * 4 + 15) & ~15u));
  uint32_t* X0 = reinterpret_cast<uint32_t*>(B0 + hsub);
  uint32_t* Y0 = X0 + hsub;
  uint32_t* Ye = Y0 + hsub;
  uint32_t(*Gs)[33] = reinterpret_cast<uint32_t(*)[33]>(Ye + hsub);
  uint16_t* outs = reinterpret_cast<uint16_t*>(Ye + hsub);  // reuses Gs after phase B
  uint32_t* H = reinterpret_cast<uint32_t*>(B0);            // block entry x group -> state (after the walks)
  DROLE(blockIdx.x, 2);
  // the bitstream is staged while the chunk CTA builds the tables: its place
  // follows from the chunk's own bytes (header size, codebook entry count);
  // the chunk CTA validates them and a disagreement restages below
  const uint64_t bit0 = static_cast<uint64_t>(b) * hbits;
  auto stage = [&](const uint8_t* bits, uint64_t nby) {
    // W[kHPre + k] = word k of the block; the two words before hold the previous block's tail
    if (b > 0) stage_bits(W, hwords, bits, nby, bit0 - 32 * kHPre);
    else {
      if (threadIdx.x < kHPre) W[threadIdx.x] = 0;
      stage_bits(W + kHPre, hwords - kHPre, bits, nby, bit0);
    }
  };
  // the block's words held in registers between issuing their loads and
  // storing them, so the loads overlap the table build (<= 3 words a thread)
  constexpr uint32_t kStageRegs = 3;
  uint32_t sw[kStageRegs];
  auto stage_issue = [&](const uint8_t* bits, uint64_t nby) {
    const int64_t byte0 = static_cast<int64_t>(bit0 >> 3) - 4 * static_cast<int64_t>(kHPre);
#pragma unroll
    for (uint32_t k = 0; k < kStageRegs; ++k) {
      const uint32_t j = threadIdx.x + k * blockDim.x;
      uint32_t v = 0;
      const int64_t bp = byte0 + 4 * static_cast<int64_t>(j);
      if (j < hwords && bp >= 0) {
        const uint64_t bb = static_cast<uint64_t>(bp);
        if (bb + 4 <= nby) {
          v = (static_cast<uint32_t>(bits[bb]) << 24) | (static_cast<uint32_t>(bits[bb + 1]) << 16) |
              (static_cast<uint32_t>(bits[bb + 2]) << 8) | bits[bb + 3];
        } else {
          for (int q = 0; q < 4; ++q) v = (v << 8) | (bb + q < nby ? bits[bb + q] : 0);
        }
      }
      sw[k] = v;
    }
  };
  auto stage_commit = [&]() {
#pragma unroll
    for (uint32_t k = 0; k < kStageRegs; ++k) {
      const uint32_t j = threadIdx.x + k * blockDim.x;
      if (j < hwords) W[j] = sw[k];
    }
  };
  // the chunk's first bytes (header, codebook of up to 64 entries) in one round
  __shared__ __align__(8) uint8_t s_hb[kLocalHdr + 8];
  __shared__ uint64_t s_vals[64], s_starts[128];
  for (uint32_t k = threadIdx.x; k < kLocalHdr; k += blockDim.x) s_hb[k] = k < hd.length ? __ldg(hd.in + k) : 0;
  __syncthreads();
  const uint64_t poff = C.payload_only ? 0 : kHeader;
  uint64_t boff = 0, nby = 0;
  if (C.length >= poff + 12) {
    boff = 12 + 5 * ld_be(s_hb + poff + 8, 4);
    if (C.length - poff >= boff) nby = C.length - poff - boff;
  }
  EMBC_DBG(const unsigned long long dt0 = dtime());
  if (hwords <= kStageRegs * blockDim.x) stage_issue(C.in + poff + boff, nby);
  else stage(C.in + poff + boff, nby);
  EMBC_DBG(__syncthreads(); const unsigned long long dt1 = dtime());
  // small calls (128-subsequence blocks) build block-local tables: there the
  // blocks start with the chunk CTAs and would otherwise wait on them
  const bool local = a.local_tables && huff_tables_local(C, s_hb, t, lut, s_vals, s_starts);
  EMBC_DBG(if (threadIdx.x == 0) {
    atomicAdd(&g_dloc[local ? 0 : 1], 1ull);
    atomicAdd(&g_dloc[2], dtime() - dt1);
    atomicAdd(&g_dloc[3], dt1 - dt0);
  });
  if (hwords <= kStageRegs * blockDim.x) stage_commit();  // read after the barriers below
  const uint64_t* vals = s_vals;
  if (!local) {
    if (threadIdx.x == 0) {  // the chunk CTA (an earlier ticket) publishes the verdict and the tables
      uint32_t delay = 32;
      while (!*reinterpret_cast<volatile uint32_t*>(&a.ready[c])) {
        __nanosleep(delay);
        delay = min(delay * 2, kPollMaxNs);
      }
      __threadfence();
      const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(&a.st[c].err);
      s_use = e == ~0ull && !*reinterpret_cast<volatile uint32_t*>(&a.hflag[c]);
    }
    __syncthreads();
    if (!s_use) {  // nothing to decode: still publish, so later blocks never wait
      if (threadIdx.x == 0) st_vol(a.blk_status + gb, kStInc | huf_state(1, 0, 0));
      return;
    }
    HView hv = hview(a.tabs, C);
    // tables written by another CTA of this launch: read through L2
    for (uint32_t i = threadIdx.x; i < (1u << kL0); i += blockDim.x) lut[i] = __ldcg(hv.lut + i);
    for (uint32_t i = threadIdx.x; i < sizeof(HTab) / 4; i += blockDim.x)
      reinterpret_cast<uint32_t*>(&t)[i] = __ldcg(reinterpret_cast<const unsigned int*>(hv.tab) + i);
    __syncthreads();
    vals = hv.vals;
    const uint64_t pay_off = __ldcg(reinterpret_cast<const unsigned long long*>(&a.st[c].pay_off));
    if (pay_off != poff || t.bit_off != boff || t.nbits != 8 * nby) {  // uniform: shared / L2 values
      stage(C.in + pay_off + t.bit_off, t.nbits / 8);
      __syncthreads();
    }
  }
  // two codewords per lookup when both fit the kL0-bit window:
  // luta = len1 | len2 << 5 | n << 10  (n: 0 long code, 1 one codeword, 2 two, 3 invalid prefix)
  for (uint32_t w = threadIdx.x; w < (1u << kL0); w += blockDim.x) {
    const uint32_t e1 = lut[w];
    uint32_t v;
    if (e1 == 0) v = 3u << 10;
    else if (e1 == kLong) v = 0;
    else {
      const uint32_t l1 = e1 & 63, rem = kL0 - l1;
      uint32_t n = 1, l2 = 0;
      if (rem) {
        const uint32_t e2 = lut[(w << l1) & ((1u << kL0) - 1)];
        if (e2 != 0 && e2 != kLong && (e2 & 63) <= rem) {
          n = 2;
          l2 = e2 & 63;
        }
      }
      v = l1 | (l2 << 5) | (n << 10);
    }
    luta[w] = static_cast<uint16_t>(v);
  }
  __syncthreads();
  DTS(blockIdx.x, 2);
  const uint32_t R = t.max_len;
  const uint64_t nbits = t.nbits;
  const uint32_t nloc = min(hsub, C.nsub - b * hsub);
  const uint32_t nent = t.nent;
  // decode from relative bit q (of subsequence i) until q >= 64, a start in
  // `stop` (the result then follows xs), or the end
  auto run = [&](uint32_t i, uint32_t q, uint64_t stop, uint32_t xs) -> uint32_t {
    const uint64_t gbase = bit0 + static_cast<uint64_t>(i) * SB;
    uint32_t n = 0;
    for (;;) {
      if (q >= SB) return pk(q - SB, 0, n);
      if ((stop >> q) & 1) return pk(pk_off(xs), pk_term(xs), n + pk_cnt(xs) - popc_below(stop, q));
      if (gbase + q >= nbits) return pk(0, 2, n);
      const uint32_t bits = speek(W, (kHPre * 32) + i * SB + q);
      const uint32_t la = luta[bits >> (32 - kL0)];
      if ((la >> 10) == 2) {
        const uint32_t l1 = la & 31, l12 = l1 + ((la >> 5) & 31);
        if (q + l1 < SB && !((stop >> (q + l1)) & 1) && gbase + q + l12 <= nbits) {
          q += l12;
          n += 2;
          continue;
        }
      }
      uint32_t len = 0;
      if (decode_one(lut, t, bits, &len) < 0) return pk(0, 1, n);
      if (gbase + q + len > nbits) return pk(0, 2, n);
      q += len;
      ++n;
    }
  };
  // ---- A.  Codes of at most 8 bits (the near-fixed-length books of the
  //      benchmarked tables among them, which self-synchronise slowly): every
  //      subsequence's full map, the state after it for each of the R entry
  //      offsets (Gs[i][16 + e]) -- the chain from offset 0 with its starts,
  //      the others until they land on one -- so the group walks below are a
  //      lookup per step.  Longer codes: a warmed-up chain per subsequence and
  //      the chain from the previous exit (A2), the walks decode the rest.
  const uint32_t i_me = threadIdx.x;
  const bool fm = R <= 8;
  if (fm) {
    if (i_me < nloc) {
      const uint64_t gbase = bit0 + static_cast<uint64_t>(i_me) * SB;
      const SubWin win(W, kHPre + SW * i_me);
      uint64_t bm = 0;
      uint32_t x0 = 0, q = 0, cnt = 0;
      for (;;) {
        if (q >= SB) {
          x0 = pk(q - SB, 0, cnt);
          break;
        }
        if (gbase + q >= nbits) {
          x0 = pk(0, 2, cnt);
          break;
        }
        const uint32_t bits = win.peek(static_cast<int>(q));
        const uint32_t la = luta[bits >> (32 - kL0)];
        if ((la >> 10) == 2) {
          const uint32_t l1 = la & 31, l12 = l1 + ((la >> 5) & 31);
          if (q + l1 < SB && gbase + q + l12 <= nbits) {
            bm |= (1ull << q) | (1ull << (q + l1));
            q += l12;
            cnt += 2;
            continue;
          }
        }
        uint32_t len = 0;
        if (decode_one(lut, t, bits, &len) < 0) {
          x0 = pk(0, 1, cnt);
          break;
        }
        if (gbase + q + len > nbits) {
          x0 = pk(0, 2, cnt);
          break;
        }
        bm |= 1ull << q;
        q += len;
        ++cnt;
      }
      Gs[i_me][16] = x0;
      for (uint32_t e = 1; e < R; ++e)
        Gs[i_me][16 + e] = ((bm >> e) & 1) ? pk(pk_off(x0), pk_term(x0), pk_cnt(x0) - popc_below(bm, e))
                                            : run(i_me, e, bm, x0);
    }
  } else {
    if (i_me < nloc) {
      const uint64_t gbase = bit0 + static_cast<uint64_t>(i_me) * SB;
      const SubWin win(W, kHPre + SW * i_me);  // the subsequence starts at word kHPre + SW i
      uint64_t bm = 0;
      uint32_t x0 = 0;
      // warm-up from 64 bits earlier (none at the very start of the stream)
      int p = gbase == 0 ? 0 : -64;
      for (;;) {
        if (p < 0) {
          const uint32_t bits = win.peek(p);
          const uint32_t la = luta[bits >> (32 - kL0)];
          if ((la >> 10) == 2 && p + static_cast<int>(la & 31) < 0) {  // both start before the subsequence
            p += static_cast<int>((la & 31) + ((la >> 5) & 31));
            continue;
          }
          uint32_t len = 0;
          if (decode_one(lut, t, bits, &len) < 0) {
            p = 0;  // the early chain died: start at the subsequence itself
            continue;
          }
          p += static_cast<int>(len);
          continue;
        }
        break;
      }
      uint32_t q = static_cast<uint32_t>(p), cnt = 0;
      for (;;) {
        if (q >= SB) {
          x0 = pk(q - SB, 0, cnt);
          break;
        }
        if (gbase + q >= nbits) {
          x0 = pk(0, 2, cnt);
          break;
        }
        const uint32_t bits = win.peek(static_cast<int>(q));
        const uint32_t la = luta[bits >> (32 - kL0)];
        if ((la >> 10) == 2) {  // two codewords, the second starting inside the subsequence
          const uint32_t l1 = la & 31, l12 = l1 + ((la >> 5) & 31);
          if (q + l1 < SB && gbase + q + l12 <= nbits) {
            bm |= (1ull << q) | (1ull << (q + l1));
            q += l12;
            cnt += 2;
            continue;
          }
        }
        uint32_t len = 0;
        if (decode_one(lut, t, bits, &len) < 0) {
          x0 = pk(0, 1, cnt);
          break;
        }
        if (gbase + q + len > nbits) {
          x0 = pk(0, 2, cnt);
          break;
        }
        bm |= 1ull << q;
        q += len;
        ++cnt;
      }
      B0[i_me] = bm;
      X0[i_me] = x0;
    }
    __syncthreads();
    if (i_me < nloc) {
      uint32_t r = 0xFFFFFFFFu, y = 0;
      if (i_me > 0 && !pk_term(X0[i_me - 1])) {
        r = pk_off(X0[i_me - 1]);
        const uint64_t bm = B0[i_me];
        const uint32_t x0 = X0[i_me];
        y = ((bm >> r) & 1) ? pk(pk_off(x0), pk_term(x0), pk_cnt(x0) - popc_below(bm, r)) : run(i_me, r, bm, x0);
      }
      Ye[i_me] = r;
      Y0[i_me] = y;
    }
  }
  __syncthreads();
  DTS(blockIdx.x, 3);
  // ---- B: group walks (Gs[i][r] = state at the entry of subsequence i for group entry r);
  //      every warp walks hsub / 8 subsequences: one group on 32 lanes, or,
  //      when codes are at most 16 (8) bits, two (four) groups of half
  //      (a quarter of) the length on 16 (8) lanes each
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lsh = R <= 8 ? 3 : (R <= 16 ? 4 : 5), lpg = 1u << lsh;  // lanes per group
  const uint32_t gpw = 32 >> lsh;
  const uint32_t gs = hsub / (8 * gpw), gsh = 31 - __clz(gs);
  const uint32_t ng = (nloc + gs - 1) >> gsh;
  if (warp * gpw < ng) {
    const uint32_t half = lane >> lsh, el = lane & (lpg - 1);
    const uint32_t g = warp * gpw + half;
    const bool gval = g < ng;
    uint32_t e = el, term = (gval && el < R) ? 0 : 3, cnt = 0;  // entries >= max_len are unreachable
    for (uint32_t j = 0; j < gs; ++j) {
      const uint32_t i = g * gs + j;
      const bool live = gval && i < nloc;
      if (live) Gs[i][el] = pk(e, term, cnt);
      uint32_t f = 0;
      if (fm) {
        if (live && !term) f = Gs[i][16 + e];  // the subsequence's full map
      } else {
        // lanes of a group that reached the same entry share one result
        const uint32_t peers = __match_any_sync(0xffffffffu, (term || !live) ? 0xFFFFFFFFu : (half << 5) | e);
        const int leader = __ffs(peers) - 1;
        if (live && !term && static_cast<int>(lane) == leader) {
          const uint64_t sbm = B0[i];
          const uint32_t sx = X0[i];
          if ((sbm >> e) & 1) f = pk(pk_off(sx), pk_term(sx), pk_cnt(sx) - popc_below(sbm, e));
          else if (Ye[i] == e) f = Y0[i];
          else f = run(i, e, sbm, sx);
        }
        f = __shfl_sync(0xffffffffu, f, leader);
      }
      if (live && !term) {
        term = pk_term(f);
        cnt += pk_cnt(f);
        e = pk_off(f);
      }
    }
    if (gval) {
      G[g][el] = pk(e, term, cnt);
      for (uint32_t x = el + lpg; x < 32; x += lpg) G[g][x] = pk(0, 3, 0);  // entries past R: unreachable
    }
  }
  __syncthreads();
  DTS(blockIdx.x, 4);
  unsigned long long* status = a.blk_status;
  if (warp == 0) {
    // lane e also records its state at every group's entry (H, over the chain
    // summaries, dead after the walks), so phase C needs no second pass
    uint32_t e = lane, term = 0, cnt = 0;
    for (uint32_t g = 0; g < ng; ++g) {
      H[g * 32 + lane] = pk(e, term, cnt);
      if (!term) {
        const uint32_t f = G[g][e];
        term = pk_term(f);
        cnt += pk_cnt(f);
        e = pk_off(f);
      }
    }
    const uint32_t bm = pk(e, term, cnt);
    BM[lane] = bm;
    a.bmaps[static_cast<uint64_t>(gb) * 32 + lane] = bm;
    __threadfence();
    __syncwarp();
    if (lane == 0 && b > 0) st_flag(status + gb, kStAgg);  // maps fenced before the warp barrier
    unsigned long long in;
    if (b == 0) {
      in = huf_state(0, 0, 0);
    } else {
      unsigned long long w;
      const uint32_t q = find_inclusive(status, C.blk0, gb, &w);
      uint32_t tm = static_cast<uint32_t>(w >> 60) & 3, ee = static_cast<uint32_t>(w >> 55) & 31;
      uint64_t cc = w & ((1ull << 55) - 1);
      // maps published after it: lane e holds entry e of each map (loads in
      // flight together), applied in order by shuffles
      for (uint32_t m0 = q + 1; m0 < gb && !tm; m0 += 8) {
        uint32_t f[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] = m0 + k < gb ? __ldcg(a.bmaps + static_cast<uint64_t>(m0 + k) * 32 + lane) : 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t v = __shfl_sync(0xffffffffu, f[k], ee);
          if (m0 + k < gb && !tm) {
            tm = pk_term(v);
            cc += pk_cnt(v);
            ee = pk_off(v);
          }
        }
      }
      in = huf_state(tm, ee, cc);
    }
    if (lane == 0) {
      uint32_t tm = static_cast<uint32_t>(in >> 60) & 3, ee = static_cast<uint32_t>(in >> 55) & 31;
      uint64_t cc = in & ((1ull << 55) - 1);
      if (!tm) {
        const uint32_t f = BM[ee];
        tm = pk_term(f);
        cc += pk_cnt(f);
        ee = pk_off(f);
      }
      st_flag(status + gb, kStInc | huf_state(tm, ee, cc));
      // fewer decodable symbols than the count: exhaustion / invalid prefix
      // (huffman.hpp:274-288) -> the exact walker reports it
      if (b == C.nblk - 1 && cc < C.N) atomicOr(&a.hflag[c], 1u);
      s_in = in;
    }
  }
  __syncthreads();
  DTS(blockIdx.x, 5);
  const uint64_t blk_base = s_in & ((1ull << 55) - 1);
  if ((s_in >> 60) & 3) return;  // the chain ended before this block
  const uint64_t N = C.N;
  if (blk_base >= N) return;
  // ---- C: decode every subsequence from its true entry
  uint32_t q = pk(0, 1, 0);
  uint64_t qbase = 0;  // index of the subsequence's first symbol
  if (threadIdx.x < nloc) {
    const uint32_t h = H[(threadIdx.x >> gsh) * 32 + (static_cast<uint32_t>(s_in >> 55) & 31)];  // group entry state
    if (!pk_term(h)) {
      q = Gs[threadIdx.x][pk_off(h)];
      qbase = blk_base + pk_cnt(h) + pk_cnt(q);
    }
  }
  __syncthreads();  // Gs is dead: its bytes take the symbols
  const bool staged = nent <= 65536;
  // per-entry output values: block-local (shared) or the chunk CTA's (global, L2)
  auto ldv = [&](uint32_t k) -> uint64_t { return local ? vals[k] : __ldcg(vals + k); };
  if (threadIdx.x < nloc && !pk_term(q)) {
    const uint32_t i = threadIdx.x;
    const uint64_t gbase = bit0 + static_cast<uint64_t>(i) * SB;
    uint64_t gi = qbase;
    uint32_t p = pk_off(q);
    const SubWin cwin(W, kHPre + SW * i);
    while (p < SB && gi < N && gbase + p < nbits) {
      const uint32_t bits = cwin.peek(static_cast<int>(p));
      if (staged && gi + 1 < N) {
        const uint32_t la = luta[bits >> (32 - kL0)];
        if ((la >> 10) == 2) {
          const uint32_t l1 = la & 31, l12 = l1 + ((la >> 5) & 31);
          if (p + l1 < SB && gbase + p + l12 <= nbits) {
            const uint32_t w = bits >> (32 - kL0);
            outs[gi - blk_base] = static_cast<uint16_t>(lut[w] >> 6);
            outs[gi + 1 - blk_base] = static_cast<uint16_t>(lut[(w << l1) & ((1u << kL0) - 1)] >> 6);
            p += l12;
            gi += 2;
            continue;
          }
        }
      }
      uint32_t len = 0;
      const int ent = decode_one(lut, t, bits, &len);
      if (ent < 0 || gbase + p + len > nbits) break;
      if (staged) {
        outs[gi - blk_base] = static_cast<uint16_t>(ent);
      } else {
        const uint64_t v = ldv(ent);
        if (C.out_kind == EMBC_OUT_F64) static_cast<uint64_t*>(C.out)[gi] = v;
        else static_cast<uint32_t*>(C.out)[gi] = static_cast<uint32_t>(v);
      }
      p += len;
      ++gi;
    }
  }
  __syncthreads();
  DTS(blockIdx.x, 6);
  if (!staged) return;
  // ---- coalesced stores of this block's symbols
  const uint32_t own = pk_cnt(BM[static_cast<uint32_t>(s_in >> 55) & 31]);
  const uint64_t nout = umin64(own, N - blk_base);
  // the decode LUT is dead now: its bytes hold the per-entry output values
  const bool f64 = C.out_kind == EMBC_OUT_F64;
  const bool vstage = nent <= (f64 ? (1u << kL0) / 2 : (1u << kL0));
  if (vstage) {
    if (f64)
      for (uint32_t k = threadIdx.x; k < nent; k += blockDim.x) reinterpret_cast<uint64_t*>(lut)[k] = ldv(k);
    else
      for (uint32_t k = threadIdx.x; k < nent; k += blockDim.x) lut[k] = static_cast<uint32_t>(ldv(k));
    __syncthreads();
  }
  if (f64) {
    uint64_t* o = static_cast<uint64_t*>(C.out) + blk_base;
    const uint64_t* sv = reinterpret_cast<const uint64_t*>(lut);
    for (uint32_t k = threadIdx.x; k < nout; k += blockDim.x) o[k] = vstage ? sv[outs[k]] : ldv(outs[k]);
  } else {
    uint32_t* o = static_cast<uint32_t*>(C.out) + blk_base;
    for (uint32_t k = threadIdx.x; k < nout; k += blockDim.x)
      o[k] = vstage ? lut[outs[k]] : static_cast<uint32_t>(ldv(outs[k]));
  }
}

// ===========================================================================
// D1 / D2
// ===========================================================================
constexpr uint32_t kDecSmem = kVlzSmem > kHuffSmem ? kVlzSmem : kHuffSmem;

// Completion counters of the decode roles: every thread fences its writes,
// then one thread counts the CTA in; waiters spin on the count.
__device__ __forceinline__ void done_signal(uint32_t* cnt) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(cnt, 1u);
}
__device__ __forceinline__ void wait_count(const uint32_t* cnt, uint32_t n) {
  uint32_t delay = 32;
  while (*reinterpret_cast<const volatile uint32_t*>(cnt) < n) {
    __nanosleep(delay);
    delay = min(delay * 2, kPollMaxNs);
  }
  __threadfence();
}

// Reference rows r0 .. r0 + nr - 1 of a vlz chunk <- their roots (V[r - r0]),
// in 16-B units when rows are 16-B aligned (else 4-B / 8-B elements); four
// units in flight per thread, all loads before the stores (a root is a
// literal row, never a destination)
__device__ void copy_ref_rows(const DChunk& C, const uint32_t* V, uint32_t r0, uint32_t nr) {
  const uint32_t D = C.dim;
  const uint32_t esz = C.out_kind == EMBC_OUT_F64 ? 8 : 4;
  const bool vec = ((D * esz) & 15) == 0 && (reinterpret_cast<uintptr_t>(C.out) & 15) == 0;
  const uint32_t upr = vec ? D * esz / 16 : D;  // units per row
  const uint32_t total = nr * upr;
  constexpr int kU = 4;
  for (uint32_t k0 = 0; k0 < total; k0 += kU * blockDim.x) {
    uint32_t ss[kU], rl[kU], cc[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t k = k0 + u * blockDim.x + threadIdx.x;
      ss[u] = 0xFFFFFFFFu;
      if (k < total) {
        rl[u] = k / upr;
        cc[u] = k - rl[u] * upr;
        const uint32_t src = V[rl[u]];
        if (src != r0 + rl[u]) ss[u] = src;
      }
    }
    if (vec) {
      uint4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (ss[u] != 0xFFFFFFFFu) v[u] = __ldcg(reinterpret_cast<const uint4*>(C.out) + static_cast<uint64_t>(ss[u]) * upr + cc[u]);
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (ss[u] != 0xFFFFFFFFu) reinterpret_cast<uint4*>(C.out)[static_cast<uint64_t>(r0 + rl[u]) * upr + cc[u]] = v[u];
    } else if (esz == 8) {
      unsigned long long v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (ss[u] != 0xFFFFFFFFu) v[u] = __ldcg(static_cast<const unsigned long long*>(C.out) + static_cast<uint64_t>(ss[u]) * upr + cc[u]);
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (ss[u] != 0xFFFFFFFFu) static_cast<unsigned long long*>(C.out)[static_cast<uint64_t>(r0 + rl[u]) * upr + cc[u]] = v[u];
    } else {
      unsigned int v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (ss[u] != 0xFFFFFFFFu) v[u] = __ldcg(static_cast<const unsigned int*>(C.out) + static_cast<uint64_t>(ss[u]) * upr + cc[u]);
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (ss[u] != 0xFFFFFFFFu) static_cast<unsigned int*>(C.out)[static_cast<uint64_t>(r0 + rl[u]) * upr + cc[u]] = v[u];
    }
  }
}

// Reference rows <- their root rows, for one tile of a vlz chunk's rows, once
// every segment of the chunk (and the roots tail) has finished.
EMBC_ROLE void copy_tile(const DecArgs& a, uint32_t b, uint8_t* smem) {
  {
    __shared__ int s_skip;
    const uint32_t c = a.ctile[3 * b];
    if (threadIdx.x == 0) {
      wait_count(&a.vdone[c], a.ch[c].nseg);
      s_skip = a.ch[c].seq || *reinterpret_cast<volatile unsigned long long*>(&a.st[c].err) != ~0ull ||
               *reinterpret_cast<volatile uint32_t*>(&a.vflag[c]);
    }
    __syncthreads();
    DTS(blockIdx.x, 2);
    if (s_skip) return;
  }
  {
    const uint32_t c = a.ctile[3 * b], r0 = a.ctile[3 * b + 1], nr = a.ctile[3 * b + 2];
    const DChunk& C = a.ch[c];
    uint32_t* src = a.row_src + C.row_base;
    // roots of the tile's rows: resolved by the chunk's last segment when its
    // row sources fit in shared memory; else pointer jumping through row_src
    // in L2, every copy tile of the chunk at once, so each round also sees the
    // other tiles' progress (a row's pointer only ever moves toward its root)
    uint32_t* V = reinterpret_cast<uint32_t*>(smem);
    if (vlz_roots_local(a, C)) {
      for (uint32_t q0 = 0; q0 < nr; q0 += 4 * blockDim.x) {
        uint32_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t r = q0 + u * blockDim.x + threadIdx.x;
          v[u] = r < nr ? __ldcg(src + r0 + r) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t r = q0 + u * blockDim.x + threadIdx.x;
          if (r < nr) V[r] = v[u];
        }
      }
      __syncthreads();
    } else {
      for (uint32_t r = threadIdx.x; r < nr; r += blockDim.x) V[r] = __ldcg(src + r0 + r);
      for (;;) {
        bool changed = false;
        for (uint32_t q0 = 0; q0 < nr; q0 += 4 * blockDim.x) {
          uint32_t v[4], vv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t r = q0 + u * blockDim.x + threadIdx.x;
            v[u] = r < nr ? V[r] : 0;
            vv[u] = (r < nr && v[u] != r0 + r) ? __ldcg(src + v[u]) : v[u];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t r = q0 + u * blockDim.x + threadIdx.x;
            if (r < nr && vv[u] != v[u]) {
              V[r] = vv[u];
              __stcg(src + r0 + r, vv[u]);
              changed = true;
            }
          }
        }
        if (!__syncthreads_or(changed)) break;
      }
    }
    DTS(blockIdx.x, 3);
    copy_ref_rows(C, V, r0, nr);
  }
}

// Per chunk, once its parallel decode has finished: the exact sequential
// walker when the chunk was planned sequential or the parallel path flagged
// it; the last chunk to finish folds the first failure into the error record.
EMBC_ROLE void finish_chunk(const DecArgs& a, uint32_t c) {
  const uint8_t codec = a.ch[c].codec;
  if (threadIdx.x == 0) {
    wait_count(&a.ready[c], 1);
    if (codec == EMBC_CODEC_VLZ && !a.ch[c].seq) wait_count(&a.vdone[c], a.ch[c].nseg);
    if (codec == EMBC_CODEC_HUFFMAN) wait_count(&a.hdone[c], a.ch[c].nblk);
    const bool ok = *reinterpret_cast<volatile unsigned long long*>(&a.st[c].err) == ~0ull;
    if (ok && ((codec == EMBC_CODEC_VLZ && (a.ch[c].seq || *reinterpret_cast<volatile uint32_t*>(&a.vflag[c]))) ||
               (codec == EMBC_CODEC_HUFFMAN && *reinterpret_cast<volatile uint32_t*>(&a.hflag[c]))))
      atomicAdd(&a.tickets[2], 1u);
  }
  __syncthreads();
  DTS(blockIdx.x, 2);
  if (codec == EMBC_CODEC_VLZ) k_dec_vlz_seq_cta(c, a.ch, a.st, nullptr, a.vflag);
  else if (codec == EMBC_CODEC_HUFFMAN) k_dec_huff_seq_cta(c, a.ch, a.st, nullptr, a.tabs, a.hflag);
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&a.tickets[1], 1u) == a.nchunks - 1;
  __syncthreads();
  if (s_last) {
    __threadfence();
    dec_fold(a.st, a.nchunks, a.err);
    if (threadIdx.x == 0) *a.diag = atomicAdd(&a.tickets[2], 0u);  // decode fallbacks of this call
    EMBC_DBG(dbg_decode_report(a));
  }
}

// One role of k_dec_main, by ticket (chunk CTAs, vlz segments, huffman
// blocks, raw tiles, copy tiles, per-chunk finishers).
__device__ __forceinline__ void dec_role(const DecArgs& a, uint32_t t, uint8_t* smem) {
  DROLE(blockIdx.x, 0);
  DTS(blockIdx.x, 1);
  if (t < a.nchunks) {  // chunk CTA: header + (huffman) decode tables, then the ready flag
    __shared__ DecState sS;
    const DChunk& C = a.ch[t];
    if (threadIdx.x == 0) {
      sS = parse_chunk(C);
      if (C.bad) {  // device-planned: the received length exceeded the chunk's capacity
        sS.err = err_key(0, EMBC_R_CAPACITY);
        sS.a = C.map_base;  // the received length
        sS.b = C.length;    // the capacity
      }
    }
    __syncthreads();
    if (C.codec == EMBC_CODEC_HUFFMAN)
      huff_tables(t, a.ch, sS, a.keys, a.tabs, a.hflag, reinterpret_cast<uint64_t*>(smem), a.smem_bytes / 8);
    __syncthreads();
    if (threadIdx.x == 0) {
      a.st[t] = sS;
      __threadfence();
      *reinterpret_cast<volatile uint32_t*>(&a.ready[t]) = 1;
    }
    DTS(blockIdx.x, 7);
    return;
  }
  t -= a.nchunks;
  const uint32_t nseg = a.dcount ? a.dcount[0] : a.nseg, nhblk = a.dcount ? a.dcount[1] : a.nhblk;
  // small calls (every role resident at once, latency-bound): the huffman
  // blocks, the longest chains, are dispatched before the vlz segments; large
  // calls keep the segments first (measured: 40.4 vs 42.3 us Kaggle-shaped,
  // 154 vs 128 us Terabyte-shaped)
  const bool hf = a.local_tables != 0;
  if (hf && t < nhblk) {
    huff_block(a, t, smem);
    DTS(blockIdx.x, 7);
    done_signal(&a.hdone[a.hblk_chunk[t]]);
    return;
  }
  if (hf) t -= nhblk;
  if (t < nseg) {
    vlz_segment(a, t, smem);
    DTS(blockIdx.x, 7);
    done_signal(&a.vdone[a.segs[t].chunk]);
    return;
  }
  t -= nseg;
  if (!hf && t < nhblk) {
    huff_block(a, t, smem);
    DTS(blockIdx.x, 7);
    done_signal(&a.hdone[a.hblk_chunk[t]]);
    return;
  }
  if (!hf) t -= nhblk;
  if (t < a.nraw) {
    DROLE(blockIdx.x, 3);
    DTS(blockIdx.x, 1);
    __shared__ DecState sR;
    const RawTile T = a.raw[t];
    const DChunk& C = a.ch[T.chunk];
    if (threadIdx.x == 0) sR = parse_chunk(C);
    __syncthreads();
    raw_tile(C, sR, T);
    DTS(blockIdx.x, 7);
    return;
  }
  t -= a.nraw;
  if (t < a.nctile) {
    DROLE(blockIdx.x, 4);
    DTS(blockIdx.x, 1);
    copy_tile(a, t, smem);
    DTS(blockIdx.x, 7);
    return;
  }
  DROLE(blockIdx.x, 5);
  DTS(blockIdx.x, 1);
  finish_chunk(a, t - a.nctile);
  DTS(blockIdx.x, 7);
}

template <bool PERSISTENT>
__global__ void __launch_bounds__(kBlock, 4) k_dec_main(DecArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t s_t;
  EMBC_DBG(if (threadIdx.x == 0 && blockIdx.x < 16384) g_cta0[blockIdx.x] = dtime());
  if constexpr (!PERSISTENT) {
    // role = block index.  Every wait is on a lower role index, and CTAs are
    // dispatched in block-index order (the same assumption as CUB's
    // single-pass scans), so a waited-on role is resident or finished.
    (void)s_t;
    const uint32_t t = blockIdx.x;
    dec_role(a, t, smem);
  } else {
    // device-planned calls: resident CTAs loop over the tickets (every wait is
    // on an earlier ticket, held by a running CTA, so the loop cannot deadlock)
    for (;;) {
      if (threadIdx.x == 0) s_t = atomicAdd(&a.tickets[0], 1u);
      __syncthreads();
      const uint32_t t = s_t;
      const uint32_t total = a.nchunks + a.dcount[0] + a.dcount[1] + a.nraw + a.nctile + a.nchunks;
      if (t >= total) return;
      dec_role(a, t, smem);
      __syncthreads();  // the role's shared state is dead before the next ticket
    }
  }
}

// Device-planned calls (embc_decode_dev): the received chunk lengths and
// offsets are device data, so the per-chunk plan the host computes for
// embc_decode (segments, blocks, table offsets) is computed here, by one CTA,
// before k_dec_main; scratch was sized by the host from the chunk capacities.
struct PlanArgs {
  DChunk* ch;
  const uint64_t* d_len;
  const uint64_t* d_off;  // may be null
  SegPair* segs;
  uint32_t* hblk_chunk;
  HBlkDesc* hblk;
  uint32_t* dcount;       // [0] vlz segments, [1] huffman blocks
  uint32_t n, hsub, sbits;
};

__global__ void __launch_bounds__(1024) k_dec_plan(PlanArgs p) {
  __shared__ unsigned long long s_tmp64[33];
  __shared__ unsigned long long s_carry[4];
  if (threadIdx.x < 4) s_carry[threadIdx.x] = 0;
  __syncthreads();
  for (uint32_t c0 = 0; c0 < p.n; c0 += blockDim.x) {
    const uint32_t c = c0 + threadIdx.x;
    unsigned long long nseg = 0, maps = 0, tabb = 0, nblk = 0;
    DChunk C{};
    if (c < p.n) {
      C = p.ch[c];
      const uint64_t cap = C.length;
      const uint64_t len = p.d_len[c];
      if (p.d_off) C.in += p.d_off[c];
      if (len > cap) {
        C.bad = 1;
        C.map_base = len;
        C.length = 0;
      } else {
        C.length = len;
      }
      const uint64_t hdr = C.payload_only ? 0 : kHeader;
      const uint64_t pay = C.length > hdr ? C.length - hdr : 0;
      if (C.bad) {
        C.seq = 1;
      } else if (C.codec == EMBC_CODEC_VLZ) {
        C.seq = (C.dim == 0 || C.dim > kVlzMaxDim || C.N >= (1ull << 31) || pay >= (1ull << 31) ||
                 (pay == 0 && C.count > 0)) ? 1 : 0;
        if (!C.seq) {
          nseg = (pay + kSeg - 1) / kSeg;
          maps = nseg * (C.dim + 1);
        }
      } else if (C.codec == EMBC_CODEC_HUFFMAN) {
        const uint64_t ecap = pay > 12 ? (pay - 12) / 5 + 1 : 1;
        uint64_t p2 = 1;
        while (p2 < ecap) p2 <<= 1;
        C.book_cap = static_cast<uint32_t>(ecap > p2 ? ecap : p2);
        const uint64_t hb = htab_bytes(C.book_cap), kb = 8 * p2 + 16;
        tabb = (hb > kb ? hb : kb);
        C.nsub = static_cast<uint32_t>((8 * (pay > 12 ? pay - 12 : 0) + p.sbits - 1) / p.sbits);
        nblk = (C.nsub + p.hsub - 1) / p.hsub;
      }
    }
    unsigned long long t0, t1, t2, t3;
    const unsigned long long e0 = block_excl_scan<unsigned long long>(nseg, s_tmp64, &t0);
    const unsigned long long e1 = block_excl_scan<unsigned long long>(maps, s_tmp64, &t1);
    const unsigned long long e2 = block_excl_scan<unsigned long long>(tabb, s_tmp64, &t2);
    const unsigned long long e3 = block_excl_scan<unsigned long long>(nblk, s_tmp64, &t3);
    if (c < p.n) {
      C.seg0 = static_cast<uint32_t>(s_carry[0] + e0);
      C.nseg = static_cast<uint32_t>(nseg);
      if (!C.bad) C.map_base = s_carry[1] + e1;
      C.tab_off = s_carry[2] + e2;
      C.blk0 = static_cast<uint32_t>(s_carry[3] + e3);
      C.nblk = static_cast<uint32_t>(nblk);
      p.ch[c] = C;
      for (uint32_t k = 0; k < nseg; ++k) p.segs[C.seg0 + k] = SegPair{c, k, C.in, static_cast<uint32_t>(C.length), C.dim};
      for (uint32_t k = 0; k < nblk; ++k) {
        p.hblk_chunk[C.blk0 + k] = c;
        p.hblk[C.blk0 + k] = HBlkDesc{c, k, C.in, C.length};
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_carry[0] += t0;
      s_carry[1] += t1;
      s_carry[2] += t2;
      s_carry[3] += t3;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    p.dcount[0] = static_cast<uint32_t>(s_carry[0]);
    p.dcount[1] = static_cast<uint32_t>(s_carry[3]);
  }
}

}  // namespace embc_dev

// ===========================================================================
// host orchestration
// ===========================================================================
namespace embc_host {

using namespace embc_dev;

static inline size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

cudaError_t decode_set_attributes() {
  cudaError_t e = cudaFuncSetAttribute(k_dec_main<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDecSmem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_dec_main<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDecSmem);
  return e;
}

// d_len == nullptr: lengths and offsets are the refs' (host plan, exact grid).
// d_len != nullptr (embc_decode_dev): refs[c].length is the chunk's capacity
// and refs[c].offset its base; the received length d_len[c] and relative
// offset d_off[c] are device data.  Scratch is sized from the capacities, the
// plan is computed on the device (k_dec_plan), and k_dec_main runs as
// persistent CTAs over the device-counted roles: no host read of the lengths,
// so the call is graph-capturable.
// Rows per copy tile: ~16384 values when the chunk's roots are resolved in
// shared memory by its last segment (the tiles only copy); larger tiles when
// they must pointer-jump through L2 themselves (each tile pays the same number
// of dependent rounds whatever its size)
static uint32_t copy_tile_rows(const embc_chunk_ref& r) {
  const uint32_t d = std::max<uint32_t>(r.dim, 1);
  const uint32_t per = std::max<uint32_t>(8, std::min<uint32_t>(4096, 16384 / d));
  if (static_cast<uint64_t>(r.count) * 4 > kDecSmem) return std::max(per, std::min<uint32_t>(4096, 131072 / d));
  return per;
}

embc_status decode(embc_ctx* ctx, const uint8_t* d_in, const embc_chunk_ref* refs, uint32_t n,
                   int out_kind, int payload_only, cudaStream_t stream, const uint64_t* d_len,
                   const uint64_t* d_off) {
  if (n == 0) return EMBC_OK;
  const bool dev = d_len != nullptr;
  if (!d_in) return set_error(ctx, EMBC_ERR_ARGUMENT, 0, 0, 0, 0, 0, "null input buffer");
  std::vector<DChunk> ch(n);
  std::vector<RawTile> raw_tiles;
  std::vector<SegPair> segs;
  std::vector<uint32_t> hblk, ctiles;
  std::vector<HBlkDesc> hdesc;
  uint64_t map_total = 0, row_total = 0, tab_total = 0, huf_subs = 0, huf_vals = 0, nseg_dev = 0;
  const uint64_t hdr = payload_only ? 0 : kHeader;
  for (uint32_t c = 0; c < n; ++c) {
    const embc_chunk_ref& r = refs[c];
    DChunk& C = ch[c];
    std::memset(&C, 0, sizeof(C));
    if (r.codec > EMBC_CODEC_HUFFMAN || (!r.out && r.count && r.dim))
      return set_error(ctx, EMBC_ERR_ARGUMENT, 0, c, 0, 0, 0, "invalid chunk reference");
    C.in = d_in + r.offset;
    C.length = r.length;
    C.out = r.out;
    C.dim = r.dim;
    C.count = r.count;
    C.N = static_cast<uint64_t>(r.dim) * r.count;
    C.eb = r.eb;
    C.codec = r.codec;
    C.payload_only = payload_only ? 1 : 0;
    C.out_kind = static_cast<uint8_t>(out_kind);
    C.fd = make_fastdiv(r.dim);
    const uint64_t pay = r.length > hdr ? r.length - hdr : 0;
    if (r.codec == EMBC_CODEC_RAW) {
      const uint64_t per = 8192;
      for (uint64_t e = 0; e < C.N; e += per) raw_tiles.push_back(RawTile{c, 0, e, std::min(per, C.N - e)});
    } else if (r.codec == EMBC_CODEC_VLZ && dev) {
      // bounds from the capacity; k_dec_plan decides seq / segments
      if (!(r.dim == 0 || r.dim > kVlzMaxDim || C.N >= (1ull << 31))) {
        const uint64_t ns = (pay + kSeg - 1) / kSeg;
        nseg_dev += ns;
        map_total += ns * (r.dim + 1);
        C.row_base = row_total;
        row_total += r.count;
        const uint32_t per = copy_tile_rows(r);
        for (uint32_t r0 = 0; r0 < r.count; r0 += per) {
          ctiles.push_back(c);
          ctiles.push_back(r0);
          ctiles.push_back(std::min(per, r.count - r0));
        }
      }
    } else if (r.codec == EMBC_CODEC_VLZ) {
      C.seq = (r.dim == 0 || r.dim > kVlzMaxDim || C.N >= (1ull << 31) || pay >= (1ull << 31) ||
               (pay == 0 && r.count > 0)) ? 1 : 0;
      if (!C.seq) {
        C.nseg = static_cast<uint32_t>((pay + kSeg - 1) / kSeg);
        C.seg0 = static_cast<uint32_t>(segs.size());
        C.map_base = map_total;
        map_total += static_cast<uint64_t>(C.nseg) * (r.dim + 1);
        C.row_base = row_total;
        row_total += r.count;
        for (uint32_t s = 0; s < C.nseg; ++s) segs.push_back(SegPair{c, s, C.in, static_cast<uint32_t>(C.length), C.dim});
        const uint32_t per = copy_tile_rows(r);
        for (uint32_t r0 = 0; r0 < r.count; r0 += per) {
          ctiles.push_back(c);
          ctiles.push_back(r0);
          ctiles.push_back(std::min(per, r.count - r0));
        }
      }
    } else {
      const uint64_t cap = pay > 12 ? (pay - 12) / 5 + 1 : 1;
      uint64_t p2 = 1;
      while (p2 < cap) p2 <<= 1;
      C.book_cap = static_cast<uint32_t>(std::max<uint64_t>(cap, p2));  // key region must hold p2
      C.tab_off = tab_total;
      tab_total += std::max<uint64_t>(htab_bytes(C.book_cap), 8 * p2 + 16);
      huf_subs += (8 * (pay > 12 ? pay - 12 : 0) + kSubBits - 1) / kSubBits;
      huf_vals += C.N;
    }
  }
  // huffman block size: 256 subsequences when there are enough for ~3 blocks per
  // SM slot, else 128 (more, shorter blocks for small calls)
  // (large calls: 16384-bit blocks of 256 x 64-bit subsequences; small calls:
  // 8192-bit blocks of 256 x 32-bit subsequences, with block-local tables)
  // (device-planned calls: by the number of values, the lengths being unknown)
  const bool small_call = dev ? huf_vals < (2ull << 20) : huf_subs < 256ull * 600;
  const uint32_t hsub = 256, sbits = small_call ? 32 : 64;
  uint64_t nhb_dev = 0;
  for (uint32_t c = 0; c < n; ++c) {
    DChunk& C = ch[c];
    if (C.codec != EMBC_CODEC_HUFFMAN) continue;
    const uint64_t pay = C.length > hdr ? C.length - hdr : 0;
    const uint32_t nsub = static_cast<uint32_t>((8 * (pay > 12 ? pay - 12 : 0) + sbits - 1) / sbits);
    if (dev) {
      nhb_dev += (nsub + hsub - 1) / hsub;
      continue;
    }
    C.nsub = nsub;
    C.nblk = (C.nsub + hsub - 1) / hsub;
    C.blk0 = static_cast<uint32_t>(hblk.size());
    for (uint32_t k = 0; k < C.nblk; ++k) {
      hblk.push_back(c);
      hdesc.push_back(HBlkDesc{c, k, C.in, C.length});
    }
  }
  if (dev && (nseg_dev >= (1ull << 31) || nhb_dev >= (1ull << 31)))
    return set_error(ctx, EMBC_ERR_UNSUPPORTED, 0, 0, 0, 0, 0, "chunk capacities beyond the device-planned decode");
  const uint32_t nseg = dev ? static_cast<uint32_t>(nseg_dev) : static_cast<uint32_t>(segs.size());
  const uint32_t nhb = dev ? static_cast<uint32_t>(nhb_dev) : static_cast<uint32_t>(hblk.size());
  const uint32_t nct = static_cast<uint32_t>(ctiles.size() / 3);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align16(off + bytes);
    return o;
  };
  const size_t o_ch = take(sizeof(DChunk) * n);
  const size_t o_raw = take(sizeof(RawTile) * (raw_tiles.size() + 1));
  const size_t o_segs = take(sizeof(SegPair) * (nseg + 1));
  const size_t o_hblk = take(sizeof(uint32_t) * (nhb + 1));
  const size_t o_hdesc = take(sizeof(HBlkDesc) * (nhb + 1));
  const size_t o_ct = take(sizeof(uint32_t) * (ctiles.size() + 1));
  const size_t o_flags = take(sizeof(uint32_t) * (6 * n + 4));  // vflag | hflag | ready | cnt | vdone | hdone | tickets
  const size_t o_sst = take(sizeof(unsigned long long) * (nseg + 1));
  const size_t o_bst = take(sizeof(unsigned long long) * (nhb + 1));
  const size_t host_bytes = off;  // uploaded (status words and flags start at zero)
  const size_t o_st = take(sizeof(DecState) * n);
  const size_t o_maps = take(sizeof(uint32_t) * (map_total + 1));
  const size_t o_bmaps = take(sizeof(uint32_t) * 32 * (nhb + 1));
  const size_t o_rsrc = take(sizeof(uint32_t) * (row_total + 1));
  const size_t o_tabs = take(tab_total + 16);
  const size_t o_keys = take(tab_total + 16);
  const size_t o_dcount = take(sizeof(uint32_t) * 4);
  cudaError_t ce = ensure_scratch(ctx, off);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "scratch allocation");
  uint8_t* hs = nullptr;
  int slot = -1;
  ce = stage_acquire(ctx, host_bytes, stream, &hs, &slot);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "staging allocation");
  std::memset(hs, 0, host_bytes);
  std::memcpy(hs + o_ch, ch.data(), sizeof(DChunk) * n);
  std::memcpy(hs + o_raw, raw_tiles.data(), sizeof(RawTile) * raw_tiles.size());
  if (!dev) {
    std::memcpy(hs + o_segs, segs.data(), sizeof(SegPair) * nseg);
    std::memcpy(hs + o_hblk, hblk.data(), sizeof(uint32_t) * nhb);
    std::memcpy(hs + o_hdesc, hdesc.data(), sizeof(HBlkDesc) * nhb);
  }
  std::memcpy(hs + o_ct, ctiles.data(), sizeof(uint32_t) * ctiles.size());
  uint8_t* d = ctx->d_scratch;
  ce = stage_upload(ctx, d, hs, host_bytes, slot, stream);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "descriptor upload");
  DecArgs a{};
  a.ch = reinterpret_cast<const DChunk*>(d + o_ch);
  a.st = reinterpret_cast<DecState*>(d + o_st);
  a.segs = reinterpret_cast<const SegPair*>(d + o_segs);
  a.hblk_chunk = reinterpret_cast<const uint32_t*>(d + o_hblk);
  a.hblk = reinterpret_cast<const HBlkDesc*>(d + o_hdesc);
  a.raw = reinterpret_cast<const RawTile*>(d + o_raw);
  a.ctile = reinterpret_cast<const uint32_t*>(d + o_ct);
  uint32_t* flags = reinterpret_cast<uint32_t*>(d + o_flags);
  a.vflag = flags;
  a.hflag = flags + n;
  a.ready = flags + 2 * n;
  a.cnt = flags + 3 * n;
  a.vdone = flags + 4 * n;
  a.hdone = flags + 5 * n;
  a.tickets = flags + 6 * n;
  a.seg_status = reinterpret_cast<unsigned long long*>(d + o_sst);
  a.blk_status = reinterpret_cast<unsigned long long*>(d + o_bst);
  a.maps = reinterpret_cast<uint32_t*>(d + o_maps);
  a.bmaps = reinterpret_cast<uint32_t*>(d + o_bmaps);
  a.row_src = reinterpret_cast<uint32_t*>(d + o_rsrc);
  a.keys = reinterpret_cast<uint64_t*>(d + o_keys);
  a.tabs = d + o_tabs;
  a.err = ctx->d_err;
  a.diag = ctx->d_diag;
  a.nchunks = n;
  a.nseg = nseg;
  a.nhblk = nhb;
  a.nraw = static_cast<uint32_t>(raw_tiles.size());
  a.nctile = nct;
  uint32_t g1 = n + nseg + nhb + a.nraw + nct + n;
  uint32_t dmax = 1;
  for (uint32_t c = 0; c < n; ++c)
    if (ch[c].codec == EMBC_CODEC_VLZ && !ch[c].seq && ch[c].dim <= kVlzMaxDim) dmax = std::max(dmax, ch[c].dim);
  a.vlz_dmax = dmax;
  a.hsub = hsub;
  a.sbits = sbits;
  a.payload_only = payload_only ? 1 : 0;
  a.local_tables = small_call ? 1 : 0;
  uint32_t smem = std::max<uint32_t>(std::max<uint32_t>(nseg ? vlz_smem(dmax) : 0, nhb ? huff_smem(hsub, sbits) : 0), 16384);
  a.smem_bytes = smem;
  if (dev) {
    PlanArgs pa{};
    pa.ch = reinterpret_cast<DChunk*>(d + o_ch);
    pa.d_len = d_len;
    pa.d_off = d_off;
    pa.segs = reinterpret_cast<SegPair*>(d + o_segs);
    pa.hblk_chunk = reinterpret_cast<uint32_t*>(d + o_hblk);
    pa.hblk = reinterpret_cast<HBlkDesc*>(d + o_hdesc);
    pa.dcount = reinterpret_cast<uint32_t*>(d + o_dcount);
    pa.n = n;
    pa.hsub = hsub;
    pa.sbits = sbits;
    EMBC_TIMED(ctx, "k_dec_plan", stream, k_dec_plan<<<1, 1024, 0, stream>>>(pa));
    a.dcount = pa.dcount;
    a.persistent = 1;
    // persistent CTAs: as many as are resident at once (never more than the roles)
    int dev_id = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev_id);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev_id);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dec_main<true>, kBlock, smem);
    g1 = std::max<uint32_t>(1, std::min<uint32_t>(g1, static_cast<uint32_t>(std::max(1, nsm * per_sm))));
  }
  if (dev) EMBC_TIMED(ctx, "k_dec_main", stream, k_dec_main<true><<<g1, kBlock, smem, stream>>>(a));
  else EMBC_TIMED(ctx, "k_dec_main", stream, k_dec_main<false><<<g1, kBlock, smem, stream>>>(a));
  ce = cudaGetLastError();
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "decode launch");
  return EMBC_OK;
}

}  // namespace embc_host
