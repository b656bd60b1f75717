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

__device__ __forceinline__ void k_dec_raw_cta(uint32_t bid, const DChunk* __restrict__ ch,
                                                    const DecState* __restrict__ st,
                                                    const RawTile* __restrict__ tiles) {
  const RawTile T = tiles[bid];
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

__device__ __forceinline__ void k_dec_vlz_seq_cta(uint32_t bid, const DChunk* __restrict__ ch, DecState* __restrict__ st,
                              const uint32_t* __restrict__ list, const uint32_t* __restrict__ vflag) {
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
// VLZ parallel decode (vlz.hpp:129-158 without its sequential dependency).
//
// A valid token stream is a sequence of "units": maximal byte runs ending in a
// byte with bit 7 clear.  Tags are one-byte units (0x00 / 0x01); every varint
// is one unit.  The token chain over units is next(u) = u + (tag ? 2 : dim+1),
// so token boundaries are recovered in parallel without side-band offsets:
//   V1 k_vlz_map    per 2 KiB byte segment: unit table, then pointer jumping
//                   gives, for each possible entry offset e in [0, dim], the
//                   exit offset into the next segment and the tokens crossed.
//   V2 k_vlz_chain  per chunk: walk the segment maps -> true entry + first row
//                   of every segment; checks the token count and the end.
//   V3 k_vlz_rows   per segment: binary lifting enumerates the chain's tags ->
//                   per row: tag unit, reference source row (offset validated).
//   V4 k_vlz_roots  per chunk: pointer jumping resolves reference chains to the
//                   root literal row.
//   V5 k_vlz_out    per element: varint of the root literal -> zigzag ->
//                   dequantize -> output tensor.
// Any anomaly flags the chunk; k_dec_vlz_seq then re-walks it sequentially to
// report the reference's exact error.
// ===========================================================================
constexpr uint32_t kSeg = 2048;        // bytes (>= units) per segment
constexpr uint32_t kVlzMaxDim = 1023;  // larger dims use the sequential walker
constexpr int kLift = 11;              // 2^11 > kSeg / 2 chain steps
constexpr uint16_t kInv = 0xFFFF;

struct SegPair {
  uint32_t chunk, seg;
};

// unit kinds: 0 = tag 0x00, 1 = tag 0x01, 2 = not a valid tag
__device__ __forceinline__ void k_vlz_map_cta(uint32_t bid, const DChunk* __restrict__ ch,
                                                    const DecState* __restrict__ st,
                                                    const SegPair* __restrict__ segs,
                                                    uint32_t* __restrict__ ustart,
                                                    uint8_t* __restrict__ ukind,
                                                    uint32_t* __restrict__ seg_units,
                                                    uint64_t* __restrict__ maps,
                                                    uint32_t* __restrict__ vflag) {
  __shared__ uint16_t J[kSeg], Cn[kSeg];
  __shared__ uint32_t uend[kSeg];
  __shared__ uint32_t s_tmp32[33];
  __shared__ int s_bad;
  const SegPair sp = segs[bid];
  const DChunk& C = ch[sp.chunk];
  if (st[sp.chunk].err != ~0ull || C.seq) return;
  const DecState& S = st[sp.chunk];
  const uint8_t* p = C.in + S.pay_off;
  const uint64_t L = S.pay_len;
  const uint32_t b0 = sp.seg * kSeg;
  const uint32_t nb = static_cast<uint32_t>(umin64(kSeg, L > b0 ? L - b0 : 0));
  const uint32_t D = C.dim;
  if (threadIdx.x == 0) s_bad = 0;
  // terminal bytes, 8 consecutive bytes per thread
  const uint32_t i0 = threadIdx.x * 8;
  uint32_t mask = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t i = i0 + k;
    if (i < nb && !(p[b0 + i] & 0x80)) mask |= 1u << k;
  }
  uint32_t U;
  uint32_t k0 = block_excl_scan<uint32_t>(__popc(mask), s_tmp32, &U);
  {
    uint32_t m = mask, k = k0;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      uend[k++] = b0 + i0 + b;
    }
  }
  __syncthreads();
  const uint64_t ubase = static_cast<uint64_t>(C.seg0 + sp.seg) * kSeg;
  for (uint32_t k = threadIdx.x; k < U; k += blockDim.x) {
    uint32_t start;
    if (k > 0) {
      start = uend[k - 1] + 1;
    } else {  // the first unit may begin in the previous segment
      start = b0;
      while (start > 0 && (p[start - 1] & 0x80) && b0 - start <= 10) --start;
    }
    const uint32_t len = uend[k] - start + 1;
    if (len > 10) s_bad = 1;  // neither a tag nor a <= 10-byte varint (bytes.hpp:139-147)
    const uint8_t v = p[start];
    const uint8_t kind = (len == 1 && v <= 1) ? v : 2;
    ustart[ubase + k] = start;
    ukind[ubase + k] = kind;
    J[k] = kind == 2 ? kInv : static_cast<uint16_t>(k + (kind == 0 ? D + 1 : 2));
    Cn[k] = 1;
  }
  // a trailing partial unit can never be consumed by a valid parse
  if (threadIdx.x == 0 && b0 + nb == L && nb > 0 && (p[L - 1] & 0x80)) s_bad = 1;
  if (threadIdx.x == 0) seg_units[C.seg0 + sp.seg] = U;
  __syncthreads();
  // pointer jumping: J[k] -> first chain unit outside the segment (or kInv),
  // Cn[k] -> tags visited from k
  for (int r = 0; r < kLift; ++r) {
    uint16_t nj[kSeg / kBlock], nc[kSeg / kBlock];
#pragma unroll
    for (uint32_t q = 0; q < kSeg / kBlock; ++q) {
      const uint32_t k = threadIdx.x + q * kBlock;
      nj[q] = 0;
      nc[q] = 0;
      if (k < U) {
        const uint16_t j = J[k];
        nj[q] = j;
        nc[q] = Cn[k];
        if (j < U) {
          nj[q] = J[j];
          nc[q] = Cn[k] + Cn[j];
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (uint32_t q = 0; q < kSeg / kBlock; ++q) {
      const uint32_t k = threadIdx.x + q * kBlock;
      if (k < U) {
        J[k] = nj[q];
        Cn[k] = nc[q];
      }
    }
    __syncthreads();
  }
  uint64_t* m = maps + C.map_base + static_cast<uint64_t>(sp.seg) * (D + 1);
  for (uint32_t e = threadIdx.x; e <= D; e += blockDim.x) {
    uint32_t exit_off, cnt;
    if (e < U) {
      const uint16_t j = J[e];
      exit_off = j == kInv ? 0xFFFFFFFFu : j - U;
      cnt = Cn[e];
    } else {
      exit_off = e - U;
      cnt = 0;
    }
    m[e] = (static_cast<uint64_t>(cnt) << 32) | exit_off;
  }
  if (threadIdx.x == 0 && s_bad) vflag[sp.chunk] = 1;
}

__device__ __forceinline__ void vlz_chain_one(const DChunk* __restrict__ ch, const DecState* __restrict__ st,
                                              uint32_t c, const uint64_t* __restrict__ maps,
                                              uint32_t* __restrict__ seg_entry, uint32_t* __restrict__ seg_row0,
                                              uint32_t* __restrict__ vflag) {
  const DChunk& C = ch[c];
  if (st[c].err != ~0ull || C.seq || vflag[c]) return;
  const uint32_t D = C.dim;
  uint32_t e = 0, row = 0;
  bool bad = false;
  for (uint32_t s = 0; s < C.nseg; ++s) {
    seg_entry[C.seg0 + s] = e;
    seg_row0[C.seg0 + s] = row;
    const uint64_t m = maps[C.map_base + static_cast<uint64_t>(s) * (D + 1) + e];
    const uint32_t exit_off = static_cast<uint32_t>(m);
    if (exit_off == 0xFFFFFFFFu) {
      bad = true;
      break;
    }
    row += static_cast<uint32_t>(m >> 32);
    e = exit_off;
    if (row > C.count) {
      bad = true;
      break;
    }
  }
  if (bad || row != C.count || e != 0) vflag[c] = 1;
}

__device__ __forceinline__ uint32_t unit_advance(const uint32_t* __restrict__ seg_units, uint32_t seg0,
                                                 uint32_t nseg, uint32_t addr, uint32_t k, bool* ok) {
  uint32_t s = addr / kSeg, l = addr % kSeg;
  while (s < nseg) {
    const uint32_t U = seg_units[seg0 + s];
    if (l + k < U) return s * kSeg + l + k;
    k -= U - l;
    l = 0;
    ++s;
  }
  *ok = false;
  return 0;
}

// varint at unit start (bytes.hpp:139-147 semantics: bits past 64 dropped)
__device__ __forceinline__ uint64_t unit_varint(const uint8_t* p, uint32_t start) {
  uint64_t v = 0;
#pragma unroll 1
  for (int shift = 0; shift < 70; shift += 7) {
    const uint8_t b = p[start++];
    if (shift < 64) v |= static_cast<uint64_t>(b & 0x7F) << shift;
    if (!(b & 0x80)) break;
  }
  return v;
}

__device__ __forceinline__ void k_vlz_rows_cta(uint32_t bid, uint8_t* dsm, const DChunk* __restrict__ ch,
                                                     const DecState* __restrict__ st,
                                                     const SegPair* __restrict__ segs,
                                                     const uint32_t* __restrict__ ustart,
                                                     const uint8_t* __restrict__ ukind,
                                                     const uint32_t* __restrict__ seg_units,
                                                     const uint32_t* __restrict__ seg_entry,
                                                     const uint32_t* __restrict__ seg_row0,
                                                     uint32_t* __restrict__ row_tag,
                                                     uint32_t* __restrict__ row_src,
                                                     uint32_t* __restrict__ vflag) {
  uint16_t (*Jt)[kSeg] = reinterpret_cast<uint16_t (*)[kSeg]>(dsm);
  const SegPair sp = segs[bid];
  const DChunk& C = ch[sp.chunk];
  if (st[sp.chunk].err != ~0ull || C.seq || vflag[sp.chunk]) return;
  const DecState& S = st[sp.chunk];
  const uint8_t* p = C.in + S.pay_off;
  const uint32_t D = C.dim;
  const uint32_t g = C.seg0 + sp.seg;
  const uint32_t U = seg_units[g];
  const uint32_t e = seg_entry[g];
  const uint32_t row0 = seg_row0[g];
  const uint32_t rowN = sp.seg + 1 < C.nseg ? seg_row0[g + 1] : C.count;
  const uint32_t T = rowN - row0;
  if (T == 0) return;
  const uint64_t ubase = static_cast<uint64_t>(g) * kSeg;
  for (uint32_t k = threadIdx.x; k < U; k += blockDim.x) {
    const uint8_t kind = ukind[ubase + k];
    Jt[0][k] = kind == 2 ? kInv : static_cast<uint16_t>(umin32(k + (kind == 0 ? D + 1 : 2), kInv - 1));
  }
  __syncthreads();
  for (int r = 1; r < kLift; ++r) {
    for (uint32_t k = threadIdx.x; k < U; k += blockDim.x) {
      const uint16_t j = Jt[r - 1][k];
      Jt[r][k] = j < U ? Jt[r - 1][j] : j;
    }
    __syncthreads();
  }
  const uint64_t rb = C.row_base;
  bool bad = false;
  for (uint32_t t = threadIdx.x; t < T; t += blockDim.x) {
    uint32_t pos = e;
    for (int r = 0; r < kLift && pos < U; ++r)
      if ((t >> r) & 1) pos = Jt[r][pos];
    if (pos >= U) {
      bad = true;
      continue;
    }
    const uint32_t row = row0 + t;
    const uint32_t addr = sp.seg * kSeg + pos;
    row_tag[rb + row] = addr;
    if (ukind[ubase + pos] == 1) {  // reference token: validate (vlz.hpp:141-145)
      bool ok = true;
      const uint32_t ga = unit_advance(seg_units, C.seg0, C.nseg, addr, 1, &ok);
      uint64_t off = 0;
      if (ok) off = unit_varint(p, ustart[static_cast<uint64_t>(C.seg0) * kSeg + ga]);
      if (!ok || off < 1 || off > row || off > kMaxWindow) {
        bad = true;
        row_src[rb + row] = row;
      } else {
        row_src[rb + row] = row - static_cast<uint32_t>(off);
      }
    } else {
      row_src[rb + row] = row;
    }
  }
  if (bad) vflag[sp.chunk] = 1;
}

constexpr uint32_t kRootSmem = 11264;  // rows resolved in shared memory (45 KiB of the stage-2 buffer)

__device__ __forceinline__ void k_vlz_roots_cta(uint32_t bid, uint8_t* dsm, const DChunk* __restrict__ ch,
                                                    const DecState* __restrict__ st,
                                                    const uint32_t* __restrict__ list,
                                                    const uint32_t* __restrict__ vflag,
                                                    uint32_t* __restrict__ row_src,
                                                    uint32_t* __restrict__ row_tag,
                                                    uint32_t* __restrict__ row_root) {
  uint32_t* sh = reinterpret_cast<uint32_t*>(dsm);
  const uint32_t c = bid;
  const DChunk& C = ch[c];
  if (st[c].err != ~0ull || C.seq || vflag[c]) return;
  const uint32_t n = C.count;
  uint32_t* src = row_src + C.row_base;
  uint32_t* a = n <= kRootSmem ? sh : src;
  if (n <= kRootSmem)
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) sh[i] = src[i];
  __syncthreads();
  for (;;) {  // pointer jumping to the root literal (every source is an earlier row)
    bool changed = false;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t s = a[i];
      const uint32_t ss = a[s];
      if (ss != s) {
        a[i] = ss;
        changed = true;
      }
    }
    if (!__syncthreads_or(changed)) break;
  }
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
    row_root[C.row_base + i] = row_tag[C.row_base + a[i]];
}

struct ElemTile {
  uint32_t chunk, pad;
  uint64_t e0, ne;
};

__device__ __forceinline__ void k_vlz_out_cta(uint32_t bid, const DChunk* __restrict__ ch,
                                                    const DecState* __restrict__ st,
                                                    const ElemTile* __restrict__ tiles,
                                                    const uint32_t* __restrict__ vflag,
                                                    const uint32_t* __restrict__ ustart,
                                                    const uint32_t* __restrict__ seg_units,
                                                    const uint32_t* __restrict__ row_root) {
  const ElemTile T = tiles[bid];
  const DChunk& C = ch[T.chunk];
  if (st[T.chunk].err != ~0ull || C.seq || vflag[T.chunk]) return;
  const DecState& S = st[T.chunk];
  const uint8_t* p = C.in + S.pay_off;
  const double w = 2.0 * S.eb;
  const uint32_t D = C.dim;
  const uint32_t* us = ustart + static_cast<uint64_t>(C.seg0) * kSeg;
  for (uint64_t e = T.e0 + threadIdx.x; e < T.e0 + T.ne; e += blockDim.x) {
    const uint32_t row = fdiv(static_cast<uint32_t>(e), C.fd);
    const uint32_t col = static_cast<uint32_t>(e) - row * D;
    bool ok = true;
    const uint32_t ga = unit_advance(seg_units, C.seg0, C.nseg, row_root[C.row_base + row], 1 + col, &ok);
    const uint64_t v = unit_varint(p, us[ga]);
    store_value(C, e, unzigzag(static_cast<uint32_t>(v)), w);
  }
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
constexpr int kL0 = 11;
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

__device__ __forceinline__ void k_huff_tables_cta(uint32_t bid, const DChunk* __restrict__ ch,
                                                        DecState* __restrict__ st,
                                                        const uint32_t* __restrict__ list,
                                                        uint64_t* __restrict__ keys,
                                                        uint8_t* __restrict__ tabs,
                                                        uint32_t* __restrict__ hflag) {
  __shared__ unsigned long long s_tmp64[33];
  __shared__ unsigned long long s_bad;
  __shared__ int s_stop;
  __shared__ HTab tb;
  const uint32_t c = list[bid];
  const DChunk C = ch[c];
  DecState& S = st[c];
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
  for (uint32_t i = threadIdx.x; i < nent; i += blockDim.x)
    hv.syms[i] = static_cast<int32_t>(static_cast<uint32_t>(key[i]) ^ 0x80000000u);
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
      hv.vals[i] = value_bits(hv.syms[i], w, C.out_kind);
    }
    carry += tot;
  }
  __syncthreads();
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
  // duplicate symbols (huffman.hpp:183-185) across all lengths
  for (uint32_t i = threadIdx.x; i < p2; i += blockDim.x)
    key[i] = i < nent ? (static_cast<uint64_t>(static_cast<uint32_t>(hv.syms[i]) ^ 0x80000000u) << 32) | i : ~0ull;
  __syncthreads();
  bitonic_sort_u64(key, p2);
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

enum : uint32_t { HF_INVALID = 1, HF_ENDED = 2, HF_DEAD = 4 };

// Decode from `pos` until crossing `end` (or the stream end / an invalid code).
__device__ __forceinline__ void decode_run(const uint8_t* s, uint64_t nbytes, uint64_t nbits,
                                           const uint32_t* lut, const HTab& t, uint64_t pos, uint64_t end,
                                           uint64_t* x, uint32_t* cnt, uint32_t* flags) {
  uint32_t c = 0, f = 0;
  while (pos < end) {
    if (pos >= nbits) {
      f |= HF_ENDED;
      break;
    }
    uint32_t len = 0;
    const int ent = decode_one(lut, t, peek32(s, nbytes, pos), &len);
    if (ent < 0) {
      f |= HF_INVALID;
      break;
    }
    if (pos + len > nbits) {
      f |= HF_ENDED;
      break;
    }
    pos += len;
    ++c;
  }
  *x = pos;
  *cnt = c;
  *flags = f;
}

struct SubTile {
  uint32_t chunk;
  uint32_t first;  // first subsequence of this CTA (multiple of kSubPerBlock)
};

constexpr uint32_t kSubPerBlock = 256;                   // subsequences per CTA / block map
constexpr uint32_t kGroup = 32;                          // subsequences per group map
constexpr uint32_t kBlockBits = kSubBits * kSubPerBlock;  // bits staged per CTA
constexpr uint32_t kStageWords = kBlockBits / 32 + 4;    // + look-ahead past the block
constexpr int kClasses = 4;                              // distinct chains tracked per subsequence
constexpr uint32_t kMapsSmem = 0;

// Packed map entry: entry/exit bit offset (5 bits) | termination kind (2 bits)
// | symbol count (25 bits).  Termination: 0 live, 1 invalid prefix, 2 stream end.
__device__ __forceinline__ uint32_t pk(uint32_t off, uint32_t term, uint32_t cnt) {
  return off | (term << 5) | (cnt << 7);
}
__device__ __forceinline__ uint32_t pk_off(uint32_t v) { return v & 31; }
__device__ __forceinline__ uint32_t pk_term(uint32_t v) { return (v >> 5) & 3; }
__device__ __forceinline__ uint32_t pk_cnt(uint32_t v) { return v >> 7; }

// Stage the CTA's slice of the bitstream as big-endian 32-bit words.
__device__ __forceinline__ void stage_bits(uint32_t* W, const uint8_t* s, uint64_t nbytes, uint64_t bit0) {
  const uint64_t b0 = bit0 >> 3;  // bit0 is a multiple of 32
  for (uint32_t w = threadIdx.x; w < kStageWords; w += blockDim.x) {
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

// 32 bits at relative bit position p of the staged words.
__device__ __forceinline__ uint32_t speek(const uint32_t* W, uint32_t p) {
  const uint32_t i = p >> 5;
  return __funnelshift_l(W[i + 1], W[i], p & 31);
}

__device__ __forceinline__ uint32_t popc_below(uint64_t bm, uint32_t p) {
  return static_cast<uint32_t>(__popcll(bm & ((1ull << p) - 1ull)));
}

// H1: for subsequence i (bits [iK, iK+K)) and each possible entry offset
// r < max_len: F_i(r) = (exit offset past (i+1)K, symbols, termination).
// Chains are decoded one after another; the codeword starts of up to
// kClasses distinct chains are kept as bitmaps in registers, and a chain that
// lands on a start of a known chain has merged with it: its result follows by
// a popcount.  (Self-synchronising codes merge within a few codewords;
// fixed-length codes need one decode per residue class.)  Groups of 32
// subsequences are then composed per entry offset (lane r), and the group maps
// per block.
__device__ __forceinline__ void k_huff_maps_cta(uint32_t bid, uint8_t* dsm, const DChunk* __restrict__ ch,
                                                             const DecState* __restrict__ st,
                                                             const SubTile* __restrict__ tiles,
                                                             uint8_t* __restrict__ tabs,
                                                             const uint32_t* __restrict__ hflag,
                                                             uint32_t* __restrict__ qmaps,
                                                             uint32_t* __restrict__ gmaps,
                                                             uint32_t* __restrict__ bmaps) {
  __shared__ HTab t;
  uint32_t* lut = reinterpret_cast<uint32_t*>(dsm);
  uint32_t* W = lut + (1 << kL0);
  uint32_t (*Fm)[33] = reinterpret_cast<uint32_t (*)[33]>(W + kStageWords);
  uint32_t (*G)[32] = reinterpret_cast<uint32_t (*)[32]>(&Fm[kSubPerBlock][0]);
  const SubTile T = tiles[bid];
  const DChunk& C = ch[T.chunk];
  if (st[T.chunk].err != ~0ull || hflag[T.chunk]) return;
  HView hv = hview(tabs, C);
  for (uint32_t i = threadIdx.x; i < (1u << kL0); i += blockDim.x) lut[i] = hv.lut[i];
  if (threadIdx.x == 0) t = *hv.tab;
  __syncthreads();
  const uint64_t bit0 = static_cast<uint64_t>(T.first) * kSubBits;
  stage_bits(W, C.in + st[T.chunk].pay_off + t.bit_off, t.nbits / 8, bit0);
  __syncthreads();
  const uint32_t R = t.max_len;
  const uint32_t sub = T.first + threadIdx.x;
  const uint64_t nbits = t.nbits;
  {
    static_assert(kSubBits == 64, "chain bitmaps are one 64-bit word");
    uint64_t cbm[kClasses];
    uint32_t cres[kClasses];
    int ncls = 0;
    const uint32_t base = threadIdx.x * kSubBits;  // relative bit of this subsequence
    for (uint32_t r = 0; r < 32; ++r) {
      uint32_t out = pk(0, 2, 0);
      if (r < R && sub < C.nsub) {
        int merged = -1;
        uint32_t mpos = 0, cnt = 0;
        uint64_t mine = 0;
        uint32_t p = r;
        for (;;) {
          if (p >= kSubBits) {
            out = pk(p - kSubBits, 0, cnt);
            break;
          }
#pragma unroll
          for (int c = 0; c < kClasses; ++c)
            if (merged < 0 && c < ncls && ((cbm[c] >> p) & 1)) merged = c;
          if (merged >= 0) {
            mpos = p;
            break;
          }
          mine |= 1ull << p;
          const uint64_t pos = bit0 + base + p;
          if (pos >= nbits) {
            out = pk(0, 2, cnt);
            break;
          }
          uint32_t len = 0;
          if (decode_one(lut, t, speek(W, base + p), &len) < 0) {
            out = pk(0, 1, cnt);
            break;
          }
          if (pos + len > nbits) {
            out = pk(0, 2, cnt);
            break;
          }
          p += len;
          ++cnt;
        }
        if (merged >= 0) {
#pragma unroll
          for (int c = 0; c < kClasses; ++c) {
            if (c == merged) {
              const uint32_t o = cres[c];
              out = pk(pk_off(o), pk_term(o), cnt + pk_cnt(o) - popc_below(cbm[c], mpos));
            }
          }
        } else if (ncls < kClasses) {
#pragma unroll
          for (int c = 0; c < kClasses; ++c) {
            if (c == ncls) {
              cbm[c] = mine;
              cres[c] = out;
            }
          }
          ++ncls;
        }
      }
      Fm[threadIdx.x][r] = out;
    }
  }
  __syncthreads();
  // group prefix maps: warp g, lane r follows entry offset r through its 32 subsequences
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t nloc = min(kSubPerBlock, C.nsub - T.first);
  {
    uint32_t e = lane, term = 0, cnt = 0;
    for (uint32_t j = 0; j < kGroup; ++j) {
      const uint32_t i = warp * kGroup + j;
      if (i < nloc) qmaps[(C.sub0 + T.first + i) * 32 + lane] = pk(e, term, cnt);
      if (!term && i < nloc) {
        const uint32_t f = Fm[i][e];
        term = pk_term(f);
        cnt += pk_cnt(f);
        e = pk_off(f);
      }
    }
    G[warp][lane] = pk(e, term, cnt);
  }
  __syncthreads();
  if (warp == 0) {  // block prefix over groups
    uint32_t e = lane, term = 0, cnt = 0;
    const uint32_t gb = static_cast<uint32_t>((C.sub0 + T.first) / kGroup);
    for (uint32_t g = 0; g < kSubPerBlock / kGroup; ++g) {
      gmaps[(gb + g) * 32 + lane] = pk(e, term, cnt);
      if (!term) {
        const uint32_t f = G[g][e];
        term = pk_term(f);
        cnt += pk_cnt(f);
        e = pk_off(f);
      }
    }
    bmaps[((C.sub0 + T.first) / kSubPerBlock) * 32 + lane] = pk(e, term, cnt);
  }
}

// H2: per chunk, walk the block maps from entry offset 0: true entry offset and
// output base of every block; then check that N symbols exist before the chain
// terminates (huffman.hpp:274-288: exhaustion / invalid prefix).
__device__ __forceinline__ void k_huff_walk_cta(uint32_t bid, uint8_t* dsm, uint32_t dsm_words, const DChunk* __restrict__ ch, const DecState* __restrict__ st,
                            const uint32_t* __restrict__ list, uint8_t* __restrict__ tabs,
                            uint32_t* __restrict__ hflag, const uint32_t* __restrict__ bmaps,
                            uint32_t* __restrict__ bentry, uint64_t* __restrict__ bbase) {
  uint32_t* sm = reinterpret_cast<uint32_t*>(dsm);
  const uint32_t c = bid;
  const DChunk& C = ch[c];
  if (st[c].err != ~0ull || hflag[c]) return;
  const uint32_t nb = (C.nsub + kSubPerBlock - 1) / kSubPerBlock;
  const uint32_t b0 = static_cast<uint32_t>(C.sub0 / kSubPerBlock);
  const bool in_smem = nb * 32 <= dsm_words;
  if (in_smem)
    for (uint32_t k = threadIdx.x; k < nb * 32; k += blockDim.x) sm[k] = bmaps[b0 * 32 + k];
  __syncthreads();
  if (threadIdx.x != 0) return;
  HView hv = hview(tabs, C);
  const uint64_t N = hv.tab->nsym;
  uint32_t e = 0, term = 0;
  uint64_t acc = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    bentry[b0 + b] = term ? 0xFFFFFFFFu : e;
    bbase[b0 + b] = acc;
    if (term) continue;
    const uint32_t m = in_smem ? sm[b * 32 + e] : bmaps[(b0 + b) * 32 + e];
    acc += pk_cnt(m);
    term = pk_term(m);
    e = pk_off(m);
  }
  // every path terminates at the stream end (term 2) unless an invalid prefix
  // comes first; either way fewer than N decodable symbols is an error
  if (acc < N) hflag[c] = 1;
}

// H3: decode every subsequence from its true start and write the values.
__device__ __forceinline__ void k_huff_out_cta(uint32_t bid, const DChunk* __restrict__ ch,
                                                           const DecState* __restrict__ st,
                                                           const SubTile* __restrict__ tiles,
                                                           uint8_t* __restrict__ tabs,
                                                           const uint32_t* __restrict__ hflag,
                                                           const uint32_t* __restrict__ qmaps,
                                                           const uint32_t* __restrict__ gmaps,
                                                           const uint32_t* __restrict__ bentry,
                                                           const uint64_t* __restrict__ bbase) {
  __shared__ uint32_t lut[1 << kL0];
  __shared__ HTab t;
  __shared__ uint32_t W[kStageWords];
  const SubTile T = tiles[bid];
  const DChunk& C = ch[T.chunk];
  if (st[T.chunk].err != ~0ull || hflag[T.chunk]) return;
  const uint32_t bidx = static_cast<uint32_t>((C.sub0 + T.first) / kSubPerBlock);
  const uint32_t be = bentry[bidx];
  if (be == 0xFFFFFFFFu) return;
  HView hv = hview(tabs, C);
  for (uint32_t i = threadIdx.x; i < (1u << kL0); i += blockDim.x) lut[i] = hv.lut[i];
  if (threadIdx.x == 0) t = *hv.tab;
  __syncthreads();
  const uint64_t bit0 = static_cast<uint64_t>(T.first) * kSubBits;
  stage_bits(W, C.in + st[T.chunk].pay_off + t.bit_off, t.nbits / 8, bit0);
  __syncthreads();
  const uint32_t sub = T.first + threadIdx.x;
  if (sub >= C.nsub) return;
  const uint32_t gidx = static_cast<uint32_t>((C.sub0 + sub) / kGroup);
  const uint32_t gm = gmaps[gidx * 32 + be];
  if (pk_term(gm)) return;
  const uint32_t qm = qmaps[(C.sub0 + sub) * 32 + pk_off(gm)];
  if (pk_term(qm)) return;
  const uint64_t base = bbase[bidx] + pk_cnt(gm) + pk_cnt(qm);
  if (base >= t.nsym) return;
  const uint32_t rel0 = threadIdx.x * kSubBits;
  uint32_t p = rel0 + pk_off(qm);
  const uint32_t end = rel0 + kSubBits;
  const uint64_t stop = t.nsym - base;
  const uint64_t nbits = t.nbits;
  const int kind = C.out_kind;
  for (uint64_t k = 0; k < stop && p < end && bit0 + p < nbits; ++k) {
    uint32_t len = 0;
    const int ent = decode_one(lut, t, speek(W, p), &len);
    if (ent < 0 || bit0 + p + len > nbits) break;
    p += len;
    const uint64_t v = hv.vals[ent];
    const uint64_t i = base + k;
    if (kind == EMBC_OUT_F64) static_cast<uint64_t*>(C.out)[i] = v;
    else static_cast<uint32_t*>(C.out)[i] = static_cast<uint32_t>(v);
  }
}

// Exact sequential walk (huffman.hpp:274-290) for flagged chunks: reproduces
// the reference's first error (exhaustion / invalid prefix / count).
__device__ __forceinline__ void k_dec_huff_seq_cta(uint32_t bid, const DChunk* __restrict__ ch, DecState* __restrict__ st,
                               const uint32_t* __restrict__ list, uint8_t* __restrict__ tabs,
                               const uint32_t* __restrict__ hflag) {
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
__device__ __forceinline__ void dec_fold(const DecState* __restrict__ st, uint32_t n, DevError* err) {
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


// ===========================================================================
// Stage kernels: every decode call is k_dec_parse + four launches.  CTAs take
// a role by blockIdx range; per-chunk follow-up work (the vlz segment-map
// walk, the reference-chain resolution, the huffman block-map walk, the
// failure fold) runs in the last CTA of its group to finish (an atomic ticket
// after a __threadfence), so it needs no launch of its own.
// ===========================================================================
struct DecPlan {
  uint32_t n_seg, n_htab, n_raw, n_sub, n_vt, nchunks;
};

struct DecArgs {
  const DChunk* ch;
  DecState* st;
  const SegPair* segs;
  const uint32_t* vlist;
  const uint32_t* hlist;
  const RawTile* raw;
  const ElemTile* vtiles;
  const SubTile* subt;
  uint32_t* vflag;
  uint32_t* hflag;
  uint32_t* cnt;  // [3][nchunks] tickets + fold ticket
  uint32_t* ustart;
  uint8_t* ukind;
  uint32_t* segu;
  uint32_t* sege;
  uint32_t* segr;
  uint64_t* maps;
  uint32_t* rtag;
  uint32_t* rsrc;
  uint32_t* rroot;
  uint64_t* keys;
  uint8_t* tabs;
  uint32_t* qmaps;
  uint32_t* gmaps;
  uint32_t* bmaps;
  uint32_t* bentry;
  uint64_t* bbase;
  DevError* err;
  uint32_t* diag;  // [0]: chunks that needed the sequential walker in this call
};

constexpr uint32_t kStage2Smem = 45312;  // max(vlz lifting tables, huffman map scratch)

__device__ __forceinline__ bool last_of(uint32_t* ticket, uint32_t total) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == total - 1;
  __syncthreads();
  if (s_last) __threadfence();
  return s_last != 0;
}

__global__ void __launch_bounds__(kBlock) k_dec_s1(DecPlan P, DecArgs a) {
  uint32_t b = blockIdx.x;
  if (b < P.n_seg) {
    k_vlz_map_cta(b, a.ch, a.st, a.segs, a.ustart, a.ukind, a.segu, a.maps, a.vflag);
    const uint32_t c = a.segs[b].chunk;
    if (last_of(&a.cnt[c], a.ch[c].nseg) && threadIdx.x == 0)
      vlz_chain_one(a.ch, a.st, c, a.maps, a.sege, a.segr, a.vflag);
    return;
  }
  b -= P.n_seg;
  if (b < P.n_htab) {
    k_huff_tables_cta(b, a.ch, a.st, a.hlist, a.keys, a.tabs, a.hflag);
    return;
  }
  b -= P.n_htab;
  k_dec_raw_cta(b, a.ch, a.st, a.raw);
}

__global__ void __launch_bounds__(kBlock) k_dec_s2(DecPlan P, DecArgs a) {
  extern __shared__ __align__(16) uint8_t dsm[];
  uint32_t b = blockIdx.x;
  if (b < P.n_seg) {
    k_vlz_rows_cta(b, dsm, a.ch, a.st, a.segs, a.ustart, a.ukind, a.segu, a.sege, a.segr, a.rtag, a.rsrc,
                   a.vflag);
    const uint32_t c = a.segs[b].chunk;
    if (last_of(&a.cnt[P.nchunks + c], a.ch[c].nseg))
      k_vlz_roots_cta(c, dsm, a.ch, a.st, nullptr, a.vflag, a.rsrc, a.rtag, a.rroot);
    return;
  }
  b -= P.n_seg;
  k_huff_maps_cta(b, dsm, a.ch, a.st, a.subt, a.tabs, a.hflag, a.qmaps, a.gmaps, a.bmaps);
  const uint32_t c = a.subt[b].chunk;
  if (last_of(&a.cnt[P.nchunks + c], (a.ch[c].nsub + kSubPerBlock - 1) / kSubPerBlock))
    k_huff_walk_cta(c, dsm, kStage2Smem / 4, a.ch, a.st, nullptr, a.tabs, a.hflag, a.bmaps, a.bentry, a.bbase);
}

__global__ void __launch_bounds__(kBlock) k_dec_s3(DecPlan P, DecArgs a) {
  const uint32_t b = blockIdx.x;
  if (b < P.n_vt) {
    k_vlz_out_cta(b, a.ch, a.st, a.vtiles, a.vflag, a.ustart, a.segu, a.rroot);
    return;
  }
  k_huff_out_cta(b - P.n_vt, a.ch, a.st, a.subt, a.tabs, a.hflag, a.qmaps, a.gmaps, a.bentry, a.bbase);
}

// Exact sequential walkers for chunks the parallel path flagged (they
// reproduce the reference's first error and message), then the fold.
__global__ void __launch_bounds__(32) k_dec_s4(DecPlan P, DecArgs a) {
  const uint32_t c = blockIdx.x;
  const uint8_t codec = a.ch[c].codec;
  if (threadIdx.x == 0 && a.st[c].err == ~0ull &&
      ((codec == EMBC_CODEC_VLZ && (a.ch[c].seq || a.vflag[c])) || (codec == EMBC_CODEC_HUFFMAN && a.hflag[c])))
    atomicAdd(a.diag, 1u);
  if (codec == EMBC_CODEC_VLZ) k_dec_vlz_seq_cta(c, a.ch, a.st, nullptr, a.vflag);
  else if (codec == EMBC_CODEC_HUFFMAN) k_dec_huff_seq_cta(c, a.ch, a.st, nullptr, a.tabs, a.hflag);
  if (last_of(&a.cnt[2 * P.nchunks], P.nchunks) && threadIdx.x == 0) dec_fold(a.st, P.nchunks, a.err);
}

}  // namespace embc_dev

namespace embc_host {
cudaError_t decode_set_attributes() {
  return cudaSuccess;
}
}  // namespace embc_host

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
  std::vector<ElemTile> vlz_tiles;
  std::vector<SegPair> segs;
  std::vector<SubTile> subtiles;
  std::vector<uint32_t> vlz_list, huf_list;
  uint64_t map_total = 0, row_total = 0, tab_total = 0, sub_total = 0;
  uint32_t seg_total = 0, max_blocks = 1;
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
    } else if (r.codec == EMBC_CODEC_VLZ) {
      vlz_list.push_back(c);
      C.seq = (r.dim == 0 || r.dim > kVlzMaxDim || C.N >= (1ull << 31) || (pay == 0 && r.count > 0)) ? 1 : 0;
      if (!C.seq) {
        C.nseg = static_cast<uint32_t>((pay + kSeg - 1) / kSeg);
        C.seg0 = seg_total;
        seg_total += C.nseg;
        C.map_base = map_total;
        map_total += static_cast<uint64_t>(C.nseg) * (r.dim + 1);
        C.row_base = row_total;
        row_total += r.count;
        for (uint32_t s = 0; s < C.nseg; ++s) segs.push_back(SegPair{c, s});
        const uint64_t per = 8192;
        for (uint64_t e = 0; e < C.N; e += per) vlz_tiles.push_back(ElemTile{c, 0, e, std::min(per, C.N - e)});
      }
    } else {
      const uint64_t cap = pay > 12 ? (pay - 12) / 5 + 1 : 1;
      uint64_t p2 = 1;
      while (p2 < cap) p2 <<= 1;
      C.book_cap = static_cast<uint32_t>(std::max<uint64_t>(cap, p2));  // key region must hold p2
      C.tab_off = tab_total;
      tab_total += std::max<uint64_t>(htab_bytes(C.book_cap), 8 * p2 + 16);
      C.nsub = static_cast<uint32_t>((8 * (pay > 12 ? pay - 12 : 0) + kSubBits - 1) / kSubBits);
      C.sub0 = sub_total;  // block-aligned so each CTA's subsequences share one block map
      sub_total += (C.nsub + kSubPerBlock - 1) / kSubPerBlock * kSubPerBlock;
      max_blocks = std::max<uint32_t>(max_blocks, (C.nsub + kSubPerBlock - 1) / kSubPerBlock);
      for (uint32_t s = 0; s < C.nsub; s += kSubPerBlock) subtiles.push_back(SubTile{c, s});
      huf_list.push_back(c);
    }
  }
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align16(off + bytes);
    return o;
  };
  const size_t o_ch = take(sizeof(DChunk) * n);
  const size_t o_raw = take(sizeof(RawTile) * (raw_tiles.size() + 1));
  const size_t o_vt = take(sizeof(ElemTile) * (vlz_tiles.size() + 1));
  const size_t o_segs = take(sizeof(SegPair) * (segs.size() + 1));
  const size_t o_st2 = take(sizeof(SubTile) * (subtiles.size() + 1));
  const size_t o_vl = take(sizeof(uint32_t) * (vlz_list.size() + 1));
  const size_t o_hl = take(sizeof(uint32_t) * (huf_list.size() + 1));
  const size_t o_flags = take(sizeof(uint32_t) * (5 * n + 1));  // vflag | hflag | tickets, zeroed by the upload
  const size_t host_bytes = off;
  const size_t o_st = take(sizeof(DecState) * n);
  const size_t o_ustart = take(sizeof(uint32_t) * (static_cast<size_t>(seg_total) * kSeg + 1));
  const size_t o_ukind = take(static_cast<size_t>(seg_total) * kSeg + 1);
  const size_t o_segu = take(sizeof(uint32_t) * (seg_total + 1));
  const size_t o_sege = take(sizeof(uint32_t) * (seg_total + 1));
  const size_t o_segr = take(sizeof(uint32_t) * (seg_total + 1));
  const size_t o_maps = take(sizeof(uint64_t) * (map_total + 1));
  const size_t o_rtag = take(sizeof(uint32_t) * (row_total + 1));
  const size_t o_rsrc = take(sizeof(uint32_t) * (row_total + 1));
  const size_t o_rroot = take(sizeof(uint32_t) * (row_total + 1));
  const size_t o_tabs = take(tab_total + 16);
  const size_t o_keys = take(tab_total + 16);
  const size_t o_pmaps = take(sizeof(uint32_t) * 32 * (sub_total + 1));
  const size_t o_gmaps = take(sizeof(uint32_t) * 32 * (sub_total / kGroup + 1));
  const size_t o_bmaps = take(sizeof(uint32_t) * 32 * (sub_total / kSubPerBlock + 1));
  const size_t o_bentry = take(sizeof(uint32_t) * (sub_total / kSubPerBlock + 1));
  const size_t o_bbase = take(sizeof(uint64_t) * (sub_total / kSubPerBlock + 1));
  cudaError_t ce = ensure_scratch(ctx, off);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "scratch allocation");
  uint8_t* hs = nullptr;
  int slot = -1;
  ce = stage_acquire(ctx, host_bytes, stream, &hs, &slot);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "staging allocation");
  std::memcpy(hs + o_ch, ch.data(), sizeof(DChunk) * n);
  std::memcpy(hs + o_raw, raw_tiles.data(), sizeof(RawTile) * raw_tiles.size());
  std::memcpy(hs + o_vt, vlz_tiles.data(), sizeof(ElemTile) * vlz_tiles.size());
  std::memcpy(hs + o_segs, segs.data(), sizeof(SegPair) * segs.size());
  std::memcpy(hs + o_st2, subtiles.data(), sizeof(SubTile) * subtiles.size());
  std::memcpy(hs + o_vl, vlz_list.data(), sizeof(uint32_t) * vlz_list.size());
  std::memcpy(hs + o_hl, huf_list.data(), sizeof(uint32_t) * huf_list.size());
  std::memset(hs + o_flags, 0, sizeof(uint32_t) * (5 * n + 1));
  uint8_t* d = ctx->d_scratch;
  ce = cudaMemcpyAsync(d, hs, host_bytes, cudaMemcpyHostToDevice, stream);
  if (ce == cudaSuccess) ce = stage_commit(ctx, slot, stream);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "descriptor upload");
  const DChunk* d_ch = reinterpret_cast<const DChunk*>(d + o_ch);
  DecState* d_st = reinterpret_cast<DecState*>(d + o_st);
  uint32_t* vflag = reinterpret_cast<uint32_t*>(d + o_flags);
  uint32_t* hflag = vflag + n;
  const uint32_t* d_vl = reinterpret_cast<const uint32_t*>(d + o_vl);
  const uint32_t* d_hl = reinterpret_cast<const uint32_t*>(d + o_hl);
  uint8_t* tabs = d + o_tabs;
  DecArgs a{};
  a.ch = d_ch;
  a.st = d_st;
  a.segs = reinterpret_cast<const SegPair*>(d + o_segs);
  a.vlist = d_vl;
  a.hlist = d_hl;
  a.raw = reinterpret_cast<const RawTile*>(d + o_raw);
  a.vtiles = reinterpret_cast<const ElemTile*>(d + o_vt);
  a.subt = reinterpret_cast<const SubTile*>(d + o_st2);
  a.vflag = vflag;
  a.hflag = hflag;
  a.cnt = vflag + 2 * n;
  a.ustart = reinterpret_cast<uint32_t*>(d + o_ustart);
  a.ukind = d + o_ukind;
  a.segu = reinterpret_cast<uint32_t*>(d + o_segu);
  a.sege = reinterpret_cast<uint32_t*>(d + o_sege);
  a.segr = reinterpret_cast<uint32_t*>(d + o_segr);
  a.maps = reinterpret_cast<uint64_t*>(d + o_maps);
  a.rtag = reinterpret_cast<uint32_t*>(d + o_rtag);
  a.rsrc = reinterpret_cast<uint32_t*>(d + o_rsrc);
  a.rroot = reinterpret_cast<uint32_t*>(d + o_rroot);
  a.keys = reinterpret_cast<uint64_t*>(d + o_keys);
  a.tabs = tabs;
  a.qmaps = reinterpret_cast<uint32_t*>(d + o_pmaps);
  a.gmaps = reinterpret_cast<uint32_t*>(d + o_gmaps);
  a.bmaps = reinterpret_cast<uint32_t*>(d + o_bmaps);
  a.bentry = reinterpret_cast<uint32_t*>(d + o_bentry);
  a.bbase = reinterpret_cast<uint64_t*>(d + o_bbase);
  a.err = ctx->d_err;
  a.diag = ctx->d_diag;
  cudaMemsetAsync(ctx->d_diag, 0, sizeof(uint32_t), stream);
  DecPlan P{};
  P.n_seg = static_cast<uint32_t>(segs.size());
  P.n_htab = static_cast<uint32_t>(huf_list.size());
  P.n_raw = static_cast<uint32_t>(raw_tiles.size());
  P.n_sub = static_cast<uint32_t>(subtiles.size());
  P.n_vt = static_cast<uint32_t>(vlz_tiles.size());
  P.nchunks = n;
  EMBC_TIMED(ctx, "k_dec_parse", stream, k_dec_parse<<<(n + 127) / 128, 128, 0, stream>>>(d_ch, d_st, n));
  if (P.n_seg + P.n_htab + P.n_raw)
    EMBC_TIMED(ctx, "k_dec_s1", stream, k_dec_s1<<<P.n_seg + P.n_htab + P.n_raw, kBlock, 0, stream>>>(P, a));
  if (P.n_seg + P.n_sub)
    EMBC_TIMED(ctx, "k_dec_s2", stream, k_dec_s2<<<P.n_seg + P.n_sub, kBlock, kStage2Smem, stream>>>(P, a));
  if (P.n_vt + P.n_sub)
    EMBC_TIMED(ctx, "k_dec_s3", stream, k_dec_s3<<<P.n_vt + P.n_sub, kBlock, 0, stream>>>(P, a));
  EMBC_TIMED(ctx, "k_dec_s4", stream, k_dec_s4<<<n, 32, 0, stream>>>(P, a));
  ce = cudaGetLastError();
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "decode launch");
  return EMBC_OK;
}

}  // namespace embc_host
