// decode.cu -- sm_100a decompression: chunk parse/validation, raw / vlz /
// huffman decoding and dequantization straight into the consumer tensor.
//
// Mirrors embc::parse_chunk + embc::decode_chunk (container.hpp:89-115,
// :146-181), vlz_decode (vlz.hpp:129-158), huff_decode (huffman.hpp:254-291),
// dequantize (quantizer.hpp:95-102).
//
// Every malformed-input check of the reference is reproduced, in the
// reference's order, so the first failure (and its message) is identical.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "embc_internal.h"

namespace embc_dev {

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
// D0: header parse (container.hpp:89-115) + metadata agreement
// (commsim.hpp:371-376) + ErrorBound (container.hpp:147, batch.hpp:33-37)
// + raw size (container.hpp:152-155).  One thread per chunk.
// ---------------------------------------------------------------------------
__global__ void k_dec_parse(const DChunk* __restrict__ ch, DecState* __restrict__ st, uint32_t n) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const DChunk C = ch[c];
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
    const uint8_t* p = C.in;
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
  st[c] = S;
}

// ---------------------------------------------------------------------------
// D1: raw payload (container.hpp:151-160): u32le codes -> values
// ---------------------------------------------------------------------------
struct RawTile {
  uint32_t chunk;
  uint32_t pad;
  uint64_t e0, ne;
};

__global__ void __launch_bounds__(kBlock) k_dec_raw(const DChunk* __restrict__ ch,
                                                    const DecState* __restrict__ st,
                                                    const RawTile* __restrict__ tiles) {
  const RawTile T = tiles[blockIdx.x];
  const DChunk& C = ch[T.chunk];
  const DecState& S = st[T.chunk];
  if (S.err != ~0ull) return;
  const uint8_t* p = C.in + S.pay_off;
  const double w = 2.0 * S.eb;
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

__global__ void k_dec_vlz_seq(const DChunk* __restrict__ ch, DecState* __restrict__ st,
                              const uint32_t* __restrict__ list) {
  if (threadIdx.x != 0) return;
  const uint32_t c = list[blockIdx.x];
  const DChunk C = ch[c];
  DecState& S = st[c];
  if (S.err != ~0ull) return;
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

// ---------------------------------------------------------------------------
// D3: huffman codebook (read_codebook + from_lengths + finalize,
// huffman.hpp:132-148, :165-186, :213-222) -- one CTA per chunk -- followed
// by the bit-serial canonical decode (huffman.hpp:254-291).
// ---------------------------------------------------------------------------
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

struct HuffTables {
  uint32_t first[33], count[33], base[33];
};

__global__ void __launch_bounds__(kBlock) k_dec_huff_seq(const DChunk* __restrict__ ch,
                                                         DecState* __restrict__ st,
                                                         const uint32_t* __restrict__ list,
                                                         uint64_t* __restrict__ keys,
                                                         int32_t* __restrict__ syms) {
  __shared__ unsigned long long s_tmp64[33];
  __shared__ unsigned long long s_bad;
  __shared__ int s_stop;
  __shared__ HuffTables tb;
  const uint32_t c = list[blockIdx.x];
  const DChunk C = ch[c];
  DecState& S = st[c];
  if (S.err != ~0ull) return;
  const uint8_t* p = C.in + S.pay_off;
  const uint64_t L = S.pay_len;
  uint64_t* key = keys + C.book_off;
  int32_t* sym = syms + C.book_off;
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
  for (uint32_t i = threadIdx.x; i < p2; i += blockDim.x) {
    if (i < nent) {
      const uint32_t s = static_cast<uint32_t>(ld_be(p + 12 + 5ull * i, 4));
      key[i] = (static_cast<uint64_t>(p[12 + 5ull * i + 4]) << 32) | (s ^ 0x80000000u);
    } else {
      key[i] = ~0ull;
    }
  }
  __syncthreads();
  bitonic_sort_u64(key, p2);
  // duplicate symbols (huffman.hpp:183-185): the map in finalize catches
  // duplicates across lengths too, so test in symbol order.
  for (uint32_t i = threadIdx.x; i < nent; i += blockDim.x) sym[i] = static_cast<int32_t>(static_cast<uint32_t>(key[i]) ^ 0x80000000u);
  if (threadIdx.x < 33) {
    tb.count[threadIdx.x] = 0;
    tb.first[threadIdx.x] = 0;
    tb.base[threadIdx.x] = 0;
  }
  __syncthreads();
  // canonical codes per length: first code of each length and its entry index
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
    }
    carry += tot;
  }
  __syncthreads();
  // duplicate check by symbol
  for (uint32_t i = threadIdx.x; i < p2; i += blockDim.x)
    key[i] = i < nent ? (static_cast<uint64_t>(static_cast<uint32_t>(sym[i]) ^ 0x80000000u) << 32) | i : ~0ull;
  __syncthreads();
  bitonic_sort_u64(key, p2);
  bool dup = false;
  for (uint32_t i = 1 + threadIdx.x; i < nent; i += blockDim.x)
    dup |= (key[i] >> 32) == (key[i - 1] >> 32);
  dup = __syncthreads_or(dup);
  if (dup) {
    if (threadIdx.x == 0) dec_fail(S, 0, EMBC_R_HUF_DUP, 0, 0);
    return;
  }
  if (threadIdx.x != 0) return;
  uint32_t max_len = 0;  // entries().back().length (huffman.hpp:257)
  for (uint32_t l = 1; l <= 32; ++l)
    if (tb.count[l]) max_len = l;
  S.max_len = max_len;
  S.bit_off = 12 + 5ull * nent;
  // bit-serial decode (huffman.hpp:274-290)
  const uint8_t* bits = p + S.bit_off;
  const uint64_t nbytes = L - S.bit_off;
  const uint64_t nsym = S.nsym;
  const double w = 2.0 * S.eb;
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
        if (i < C.N) store_value(C, i, sym[tb.base[len] + (code - tb.first[len])], w);
        break;
      }
      if (len >= max_len) {
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
__global__ void k_dec_fold(const DecState* __restrict__ st, uint32_t n, DevError* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (uint32_t c = 0; c < n; ++c) {
    const DecState& S = st[c];
    if (S.err == ~0ull) continue;
    if (err->valid) return;
    err->valid = 1;
    err->job = c;
    err->reason = static_cast<int32_t>(S.err & 63);
    err->index = S.err >> 6;
    err->a = S.a;
    err->b = S.b;
    err->eb = S.eb;
    const int r = err->reason;
    err->status = (r == EMBC_R_BAD_EB) ? EMBC_ERR_VALUE
                  : (r == EMBC_R_RANGE) ? EMBC_ERR_UNSUPPORTED
                                        : EMBC_ERR_FORMAT;
    return;
  }
}

}  // namespace embc_dev

// ===========================================================================
// host orchestration
// ===========================================================================
namespace embc_host {

using namespace embc_dev;

static inline size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

embc_status decode(embc_ctx* ctx, const uint8_t* d_in, const embc_chunk_ref* refs, uint32_t n,
                   int out_kind, int payload_only, cudaStream_t stream) {
  if (n == 0) return EMBC_OK;
  if (!d_in) return set_error(ctx, EMBC_ERR_ARGUMENT, 0, 0, 0, 0, 0, "null input buffer");
  std::vector<DChunk> ch(n);
  std::vector<RawTile> raw_tiles;
  std::vector<uint32_t> vlz_list, huf_list;
  uint64_t book_total = 0;
  uint32_t max_p2 = 1;
  for (uint32_t c = 0; c < n; ++c) {
    const embc_chunk_ref& r = refs[c];
    DChunk& C = ch[c];
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
    C.book_off = 0;
    C.book_cap = 0;
    if (r.codec == EMBC_CODEC_RAW) {
      const uint64_t per = 8192;
      for (uint64_t e = 0; e < C.N; e += per) raw_tiles.push_back(RawTile{c, 0, e, std::min(per, C.N - e)});
    } else if (r.codec == EMBC_CODEC_VLZ) {
      vlz_list.push_back(c);
    } else {
      const uint64_t hdr = payload_only ? 0 : kHeader;
      const uint64_t cap = r.length > hdr + 12 ? (r.length - hdr - 12) / 5 + 1 : 1;
      uint32_t p2 = 1;
      while (p2 < cap) p2 <<= 1;
      C.book_off = static_cast<uint32_t>(book_total);
      C.book_cap = static_cast<uint32_t>(cap);
      book_total += p2;
      max_p2 = std::max(max_p2, p2);
      huf_list.push_back(c);
    }
  }
  size_t off = 0;
  const size_t o_ch = off;
  off = align16(off + sizeof(DChunk) * n);
  const size_t o_raw = off;
  off = align16(off + sizeof(RawTile) * (raw_tiles.size() + 1));
  const size_t o_vl = off;
  off = align16(off + sizeof(uint32_t) * (vlz_list.size() + 1));
  const size_t o_hl = off;
  off = align16(off + sizeof(uint32_t) * (huf_list.size() + 1));
  const size_t host_bytes = off;
  const size_t o_st = off;
  off = align16(off + sizeof(DecState) * n);
  const size_t o_keys = off;
  off = align16(off + sizeof(uint64_t) * (book_total + 1));
  const size_t o_syms = off;
  off = align16(off + sizeof(int32_t) * (book_total + 1));
  cudaError_t ce = ensure_scratch(ctx, off);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "scratch allocation");
  uint8_t* hs = nullptr;
  int slot = -1;
  ce = stage_acquire(ctx, host_bytes, stream, &hs, &slot);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "staging allocation");
  std::memcpy(hs + o_ch, ch.data(), sizeof(DChunk) * n);
  std::memcpy(hs + o_raw, raw_tiles.data(), sizeof(RawTile) * raw_tiles.size());
  std::memcpy(hs + o_vl, vlz_list.data(), sizeof(uint32_t) * vlz_list.size());
  std::memcpy(hs + o_hl, huf_list.data(), sizeof(uint32_t) * huf_list.size());
  uint8_t* d = ctx->d_scratch;
  ce = cudaMemcpyAsync(d, hs, host_bytes, cudaMemcpyHostToDevice, stream);
  if (ce == cudaSuccess) ce = stage_commit(ctx, slot, stream);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "descriptor upload");
  const DChunk* d_ch = reinterpret_cast<const DChunk*>(d + o_ch);
  DecState* d_st = reinterpret_cast<DecState*>(d + o_st);
  EMBC_TIMED(ctx, "k_dec_parse", stream, k_dec_parse<<<(n + 127) / 128, 128, 0, stream>>>(d_ch, d_st, n));
  if (!raw_tiles.empty())
    EMBC_TIMED(ctx, "k_dec_raw", stream, k_dec_raw<<<static_cast<uint32_t>(raw_tiles.size()), kBlock, 0, stream>>>(
        d_ch, d_st, reinterpret_cast<const RawTile*>(d + o_raw)));
  if (!vlz_list.empty())
    EMBC_TIMED(ctx, "k_dec_vlz_seq", stream, k_dec_vlz_seq<<<static_cast<uint32_t>(vlz_list.size()), 32, 0, stream>>>(
        d_ch, d_st, reinterpret_cast<const uint32_t*>(d + o_vl)));
  if (!huf_list.empty())
    EMBC_TIMED(ctx, "k_dec_huff_seq", stream, k_dec_huff_seq<<<static_cast<uint32_t>(huf_list.size()), kBlock, 0, stream>>>(
        d_ch, d_st, reinterpret_cast<const uint32_t*>(d + o_hl),
        reinterpret_cast<uint64_t*>(d + o_keys), reinterpret_cast<int32_t*>(d + o_syms)));
  EMBC_TIMED(ctx, "k_dec_fold", stream, k_dec_fold<<<1, 32, 0, stream>>>(d_st, n, ctx->d_err));
  ce = cudaGetLastError();
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "decode launch");
  return EMBC_OK;
}

}  // namespace embc_host
