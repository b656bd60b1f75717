// encode.cu -- sm_100a compression pipeline: quantize -> (vlz dedup | huffman
// | raw) -> chunk container -> packed send buffer, for a batch of jobs in TWO
// launches with no host synchronisation (graph-capturable).
//
// Mirrors embc::encode_chunks + embc::pack (container.hpp:119-142, :242-256,
// :304-311).  Kernels:
//   E1 k_stats   one CTA per tile: 128-bit loads, quantize (quantizer.hpp:43-76),
//                first-failure key, code range + warp-aggregated histogram
//                (huffman jobs, Codebook::build huffman.hpp:122-128), per-row
//                hash + literal token length (vlz jobs, vlz.hpp:115-118).  The
//                last tile of a huffman job to finish builds its canonical
//                codebook (huffman.hpp:49-120, :165-186) in the same launch.
//   E2 k_emit    one CTA per tile, tiles taken in order from an atomic ticket:
//                vlz match decisions (vlz.hpp:86-103) / huffman bit counts /
//                raw sizes, then a decoupled look-back over tiles (offsets
//                inside a chunk) and over jobs (chunk offsets in job order,
//                container.hpp:245-250), then the bytes: tokens / MSB-first
//                bitstream (bitstream.hpp:32-51) / u32le codes, chunk headers,
//                pack table and 25-B metadata written by each job's last tile.
#include <cuda_runtime.h>
#include <limits.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "embc_internal.h"

namespace embc_dev {

#include "encode_timeline.cuh"  // EMBC_DEBUG builds only: per-phase device timestamps

constexpr uint32_t kTileVals = 4096;     // values per tile (whole rows): 3 CTAs of E2 per SM
constexpr uint32_t kMaxRowVals = 8192;   // a single row (dim) may exceed kTileVals up to this
constexpr uint32_t kMaxTileRows = 1024;  // rows per tile (bounds the per-row smem arrays)
constexpr uint32_t kHashStage = 2048;    // vlz: row hashes of [row0 - W, row0 + rows) staged in smem
constexpr uint32_t kLutStage = 2048;     // huffman: codebook LUT entries staged in smem
constexpr uint32_t kSmemBook = 1024;     // codebook symbols sorted fully in shared memory

// E2 dynamic shared memory carve (bytes) for tiles of <= vals values / rows rows:
//   [codes: padded, rows*(dim|1) or l + l/32][stage: output bytes][aux: hashes + dec/lit | LUT]
__host__ __device__ constexpr uint32_t emit_codes_bytes(uint32_t vals, uint32_t rows) {
  // vlz / raw: vals (row-major); huffman: l + l/32 padding
  return (((vals + vals / 32 + 64) * 4 + 15) & ~15u) + 0 * rows;
}
__host__ __device__ constexpr uint32_t emit_stage_bytes(uint32_t vals, uint32_t rows, bool vlz = true) {
  return ((vlz ? rows + 5 * vals : 4 * vals) + 128 + 15) & ~15u;
}
constexpr uint32_t kAuxBytes = kHashStage * 4 + kMaxTileRows * 20 + 8 * kLutStage;  // LUT / hash stage | per-row arrays
constexpr uint32_t kEmitSmemMax = emit_codes_bytes(kMaxRowVals, kMaxTileRows) +
                                  emit_stage_bytes(kMaxRowVals, kMaxTileRows) + kAuxBytes;
// E1: codes staged for the generic (scalar) path + histogram window; the
// codebook tail reuses the same bytes (>= kSmemBook * 32)
__host__ __device__ constexpr uint32_t stats_codes_bytes(uint32_t vals, uint32_t rows) {
  return (vals + rows) * 4 > 16384 ? ((vals + rows) * 4 + 15) & ~15u : 16384u;
}
constexpr uint32_t kTileHist = 256;  // bins of a huffman tile's kept histogram (two-pass calls)
constexpr uint32_t kStatsVlzAux = 4 * kHashStage + 16 * kMaxTileRows + 4 * 2048 + 2 * kHashStage;
constexpr uint32_t kEncodeSmemMax = 200 * 1024;  // k_encode (merged E1 + E2): picked per call when it fits
constexpr uint32_t kStatsSmemMax =
    stats_codes_bytes(kMaxRowVals, kMaxTileRows) + (kWin * 4 > kStatsVlzAux ? kWin * 4 : kStatsVlzAux);

// look-back status words: flag in bits 63:62, value in 61:0
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;
constexpr uint32_t kJobStride = 16;  // job status words one 128-B line apart (polled by many CTAs)

// call-level flags (device): [0] abort bits, [1] E2 tile ticket, [2..3] wide-pool cursor (u64)
enum : uint32_t { CF_ABORT = 0, CF_TICKET = 1, CF_WIDE = 2, CF_TICKET_S = 4 };

// ---------------------------------------------------------------------------
// element access (int32 code sources for the codec-stage entry points)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int32_t job_code(const DJob& J, uint64_t e, uint32_t* reason) {
  if (J.src_kind == EMBC_SRC_F32) {
    const float x = __ldg(static_cast<const float*>(J.src) + e);
    return quantize_f32(x, J.qp, reason);
  }
  return __ldg(static_cast<const int32_t*>(J.src) + e);
}

// Row hash: sum_j code_j * K(j) mod 2^32 with pseudo-random odd per-column
// multipliers, so partial sums combine in any order (warp shuffles) at one
// IMAD per element.  Equality is verified exactly (CodeRowEq, vlz.hpp:75-79),
// so only the hit rate depends on the function.
__device__ __forceinline__ uint32_t col_key(uint32_t col) {
  uint32_t x = col * 0x9E3779B1u + 0x7F4A7C15u;
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x | 1u;
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long n = __shfl_xor_sync(0xffffffffu, v, o);
    v = n < v ? n : v;
  }
  return v;
}

// warp-aggregated histogram increment: lanes with equal bins add once
__device__ __forceinline__ void hist_add(uint32_t* shist, uint32_t bin) {
  const uint32_t peers = __match_any_sync(0xffffffffu, bin);
  const uint32_t lane = threadIdx.x & 31;
  if (bin != 0xFFFFFFFFu && (__ffs(peers) - 1) == static_cast<int>(lane)) atomicAdd(&shist[bin], __popc(peers));
}

__device__ __forceinline__ uint32_t ld_u32_cg(const void* p) { return __ldcg(static_cast<const unsigned int*>(p)); }

// ---------------------------------------------------------------------------
// Canonical Huffman codebook of one job (run by the job's last E1 tile).
// ---------------------------------------------------------------------------
// In-place ascending bitonic sort of p2 keys (shared or global memory).
__device__ void bitonic_sort(uint64_t* key, uint32_t p2) {
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

struct BookScratch {
  uint64_t* key;    // p2 entries
  uint64_t* wgt;    // 2 * cap (leaf + merged weights)
  int32_t* parent;  // 2 * cap
};

struct BookArgs {
  uint32_t* hist;       // [nhuff windows | wide pool]
  uint64_t* lut;        // mirrors hist: (codeword << 8 | length) per code
  uint8_t* books;       // serialized codebooks (write_codebook, huffman.hpp:202-209)
  uint64_t book_stride;
  BookScratch gs;       // global sort scratch for alphabets > kSmemBook
  uint64_t gs_stride;
  uint32_t nhuff;
  uint32_t* flags;      // call flags
};

// Codebook of an alphabet of <= 256 symbols by one warp: the same steps as the
// block version below (huffman.hpp:49-120 lengths, :165-186 canonical codes).
// Ascending sort of n <= 64 distinct keys in shared memory by one warp: each
// lane ranks its (up to) two keys against all n, then scatters.
__device__ __forceinline__ void warp_rank_sort64(uint64_t* key, uint32_t n) {
  const uint32_t lane = threadIdx.x & 31;
  uint64_t k0 = lane < n ? key[lane] : 0, k1 = lane + 32 < n ? key[lane + 32] : 0;
  uint32_t r0 = 0, r1 = 0;
#pragma unroll 4
  for (uint32_t j = 0; j < n; ++j) {
    const uint64_t kj = key[j];
    r0 += kj < k0 ? 1u : 0u;
    r1 += kj < k1 ? 1u : 0u;
  }
  __syncwarp();
  if (lane < n) key[r0] = k0;
  if (lane + 32 < n) key[r1] = k1;
  __syncwarp();
}

__device__ void book_warp(const DJob& J, JobState* Sp, const BookArgs& a, uint64_t* key, uint64_t* wgt,
                          int32_t* parent, uint32_t nsym, uint32_t p2, uint32_t* gh, uint64_t span, int32_t cmin,
                          uint64_t* L, uint8_t* book, uint64_t lut_off) {
  const uint32_t lane = threadIdx.x & 31;
  // 2. leaves sorted by (count, symbol) (huffman.hpp:74-77); keys are distinct
  if (nsym > 1) {
    if (nsym <= 64) warp_rank_sort64(key, nsym);
    else warp_sort_smem(key, p2);
  }
  TS1(8);
  // 3. two-queue merge, leaf queue preferred on ties (huffman.hpp:91-109);
  //    weights are symbol counts and their sums (< 2^32 values per chunk)
  uint32_t* w32 = reinterpret_cast<uint32_t*>(wgt);
  for (uint32_t i = lane; i < nsym; i += 32) w32[i] = static_cast<uint32_t>(key[i] >> 32);
  __syncwarp();
  if (nsym > 1 && lane == 0) {
    // the merged queue's weights are created in non-decreasing order; three
    // heads of each queue live in registers (wl_k == w32[lh + k] while
    // lh + k < n, wm_k == w32[mh + k] while mh + k < size) and each pick
    // loads the head three places on, so no load is on the chain; a merged
    // head not yet created is set from the new node's weight when it is
    const uint32_t n = nsym, total = 2 * n - 1;
    uint32_t size = n, lh = 0, mh = n;
    uint32_t wl0 = w32[0], wl1 = w32[min(1u, n - 1)], wl2 = w32[min(2u, n - 1)], wm0 = 0, wm1 = 0, wm2 = 0;
    while (size < total) {
      uint32_t ab[2];
      uint32_t w2 = 0;
#pragma unroll
      for (int k = 0; k < 2; ++k) {  // branch-free pick: selects, loads issued unconditionally
        const bool tl = lh < n && (mh >= size || wl0 <= wm0);
        ab[k] = tl ? lh : mh;
        w2 += tl ? wl0 : wm0;
        lh += tl ? 1u : 0u;
        mh += tl ? 0u : 1u;
        const uint32_t ln = w32[min(lh + 2, n - 1)];
        const uint32_t mn = w32[min(mh + 2, total - 1)];
        wl0 = tl ? wl1 : wl0;
        wl1 = tl ? wl2 : wl1;
        wl2 = tl ? ln : wl2;
        wm0 = tl ? wm0 : wm1;
        wm1 = tl ? wm1 : wm2;
        wm2 = tl ? wm2 : mn;
      }
      w32[size] = w2;
      const uint32_t d = size - mh;  // the new node's place among the merged heads
      wm0 = d == 0 ? w2 : wm0;
      wm1 = d == 1 ? w2 : wm1;
      wm2 = d == 2 ? w2 : wm2;
      parent[ab[0]] = static_cast<int32_t>(size);
      parent[ab[1]] = static_cast<int32_t>(size);
      ++size;
    }
    parent[total - 1] = -1;
  }
  __syncwarp();
  TS1(9);
  // 4. lengths = leaf depth; the first leaf (sorted order) past 32 bits fails (huffman.hpp:110-118)
  //    Each lane walks two leaves' parent chains side by side.
  unsigned long long cap = ~0ull, bits = 0;
  for (uint32_t i0 = 0; i0 < nsym; i0 += 64) {
    const uint32_t ia = i0 + lane, ib = ia + 32;
    uint32_t da = 0, db = 0;
    if (nsym == 1) {
      da = 1;
    } else {
      int32_t qa = ia < nsym ? parent[ia] : -1, qb = ib < nsym ? parent[ib] : -1;
      while ((qa & qb) != -1) {  // either chain still below the root
        const int32_t na = parent[qa < 0 ? 0 : qa], nb = parent[qb < 0 ? 0 : qb];
        da += qa != -1 ? 1u : 0u;
        db += qb != -1 ? 1u : 0u;
        qa = qa != -1 ? na : -1;
        qb = qb != -1 ? nb : -1;
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t i = h ? ib : ia, depth = h ? db : da;
      if (i >= nsym) continue;
      if (depth > 32) cap = min(cap, (static_cast<unsigned long long>(i) << 32) | depth);
      bits += (key[i] >> 32) * depth;  // count x code length: the payload bits
      key[i] = (static_cast<uint64_t>(depth > 32 ? 63 : depth) << 32) | (key[i] & 0xFFFFFFFFull);
    }
  }
  cap = warp_min_u64(cap);
  if (cap != ~0ull) {
    if (lane == 0) {
      Sp->aux = cap & 0xFFFFFFFFull;
      atomicMin(reinterpret_cast<unsigned long long*>(&Sp->err), err_key(cap >> 32, EMBC_R_HUF_LEN_CAP) | (1ull << 63));
      atomicOr(&a.flags[CF_ABORT], JF_ABORT);
    }
    for (uint64_t b = lane; b < span; b += 32) gh[b] = 0;
    return;
  }
  __syncwarp();
  TS1(10);
  // 5. canonical order (length asc, symbol asc); keys are distinct
  if (nsym > 1) {
    if (nsym <= 64) warp_rank_sort64(key, nsym);
    else warp_sort_smem(key, p2);
  }
  TS1(11);
  // 6. canonical codes: code_i = sum_{j<i} 2^(len_i - len_j) (finalize, huffman.hpp:170-181)
  unsigned long long carry = 0;
  for (uint32_t i0 = 0; i0 < nsym; i0 += 32) {
    const uint32_t i = i0 + lane;
    uint32_t len = 0, symoff = 0;
    unsigned long long kraft = 0;
    if (i < nsym) {
      len = static_cast<uint32_t>(key[i] >> 32);
      symoff = static_cast<uint32_t>(key[i]);
      kraft = 1ull << (32 - len);
    }
    const unsigned long long inc = warp_incl_scan<unsigned long long>(kraft);
    if (i < nsym) {
      const uint64_t prefix = carry + inc - kraft;
      const uint32_t cw = static_cast<uint32_t>(prefix >> (32 - len));
      L[symoff] = (static_cast<uint64_t>(cw) << 8) | len;
      uint8_t* e = book + 12 + 5ull * i;
      st_be(e, static_cast<uint32_t>(static_cast<int32_t>(static_cast<int64_t>(cmin) + symoff)), 4);
      e[4] = static_cast<uint8_t>(len);
    }
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  bits = warp_sum<unsigned long long>(bits);
  __syncwarp();
  for (uint64_t b = lane; b < span; b += 32) gh[b] = 0;  // clean for the next call
  if (lane == 0) {
    st_be(book, J.N, 8);       // u64be symbol_count (huffman.hpp:203)
    st_be(book + 8, nsym, 4);  // u32be entry_count (huffman.hpp:204)
    Sp->nsym = nsym;
    Sp->bits = bits;
    Sp->lut_off = lut_off;
    Sp->payload = 12 + 5ull * nsym + (bits + 7) / 8;
  }
}

__device__ void build_book(const DJob& J, JobState* Sp, const BookArgs& a, uint8_t* smem) {
  __shared__ uint32_t s_tmp32[33];
  __shared__ unsigned long long s_tmp64[33];
  __shared__ unsigned long long s_cap;
  __shared__ unsigned long long s_woff;
  __shared__ int s_cmin, s_cmax, s_wide;
  __shared__ unsigned long long s_err;
  const uint32_t hj = static_cast<uint32_t>(J.hjob);
  uint32_t* narrow = a.hist + static_cast<uint64_t>(hj) * kWin;
  if (threadIdx.x == 0) {  // state written by other CTAs' atomics: read through L2
    s_err = __ldcg(reinterpret_cast<const unsigned long long*>(&Sp->err));
    s_cmin = static_cast<int>(ld_u32_cg(&Sp->cmin));
    s_cmax = static_cast<int>(ld_u32_cg(&Sp->cmax));
    s_wide = static_cast<int>(ld_u32_cg(&Sp->wide));
  }
  __syncthreads();
  if (s_err != ~0ull || J.N == 0) {
    // quantization failed (or nothing to code): leave the window histogram clean
    for (uint32_t b = threadIdx.x; b < kWin; b += blockDim.x) narrow[b] = 0;
    if (J.N == 0 && s_err == ~0ull && threadIdx.x == 0) {  // huffman.hpp:229
      Sp->err = err_key(0, EMBC_R_HUF_EMPTY) | (1ull << 63);
      atomicOr(&a.flags[CF_ABORT], JF_ABORT);
    }
    return;
  }
  TS1(5);
  const int32_t cmin = s_cmin;
  const uint64_t span = static_cast<uint64_t>(static_cast<int64_t>(s_cmax) - cmin + 1);
  uint32_t* gh;
  uint64_t lut_off;
  if (s_wide) {
    // alphabet wider than the E1 window: histogram over [cmin, cmax] in the
    // wide pool (huffman.hpp:122-128), EMBC_R_RANGE beyond kHistCap
    for (uint32_t b = threadIdx.x; b < kWin; b += blockDim.x) narrow[b] = 0;
    if (threadIdx.x == 0) {
      s_woff = ~0ull;
      if (span <= kHistCap) {
        const unsigned long long o =
            atomicAdd(reinterpret_cast<unsigned long long*>(a.flags + CF_WIDE), static_cast<unsigned long long>(span));
        if (o + span <= kWidePool) s_woff = o;
      }
    }
    __syncthreads();
    if (s_woff == ~0ull) {
      if (threadIdx.x == 0) {
        Sp->aux = span;
        Sp->err = err_key(0, EMBC_R_RANGE) | (1ull << 63);
        atomicOr(&a.flags[CF_ABORT], JF_ABORT);
      }
      return;
    }
    gh = a.hist + static_cast<uint64_t>(a.nhuff) * kWin + s_woff;
    for (uint64_t e = threadIdx.x; e < J.N; e += blockDim.x) {
      uint32_t r = 0;
      atomicAdd(&gh[job_code(J, e, &r) - cmin], 1u);
    }
    __threadfence();
    __syncthreads();
    lut_off = static_cast<uint64_t>(a.nhuff) * kWin + s_woff;
  } else {
    gh = narrow + (cmin + static_cast<int32_t>(kWin / 2));
    lut_off = static_cast<uint64_t>(hj) * kWin + (cmin + static_cast<int32_t>(kWin / 2));
  }

  // 1. nonzero bins -> symbols in ascending order (sorted histogram, huffman.hpp:51)
  //    as (count << 32 | sym - cmin) keys; one pass when the span alone bounds
  //    the symbols to the shared-memory sort, else a counting pass first
  uint32_t nsym = 0;
  if (span > kSmemBook) {
    uint32_t cnt = 0;
    for (uint64_t b = threadIdx.x; b < span; b += blockDim.x) cnt += __ldcg(gh + b) != 0;
    nsym = block_sum<uint32_t>(cnt, s_tmp32);
  }
  TS1(6);
  const bool in_smem = span <= kSmemBook || nsym <= kSmemBook;
  uint64_t* key = in_smem ? reinterpret_cast<uint64_t*>(smem) : a.gs.key + hj * a.gs_stride;
  uint64_t* wgt = in_smem ? key + kSmemBook : a.gs.wgt + hj * 2 * a.gs_stride;
  int32_t* parent = in_smem ? reinterpret_cast<int32_t*>(wgt + 2 * kSmemBook) : a.gs.parent + hj * 2 * a.gs_stride;
  {
    uint64_t base = 0;
    for (uint64_t b0 = 0; b0 < span; b0 += blockDim.x) {
      const uint64_t b = b0 + threadIdx.x;
      const uint32_t c = b < span ? __ldcg(gh + b) : 0;
      uint32_t tot;
      const uint32_t pos = block_excl_scan<uint32_t>(c != 0, s_tmp32, &tot);
      if (c) key[base + pos] = (static_cast<uint64_t>(c) << 32) | b;
      base += tot;
    }
    nsym = static_cast<uint32_t>(base);
  }
  uint32_t p2 = 1;
  while (p2 < nsym) p2 <<= 1;
  for (uint32_t i = nsym + threadIdx.x; i < p2; i += blockDim.x) key[i] = ~0ull;
  __syncthreads();
  uint8_t* book = a.books + hj * a.book_stride;
  uint64_t* L = a.lut + lut_off;
  TS1(7);
  TS1V(12, nsym);
  TS1V(13, span);
  if (p2 <= 256 && in_smem) {  // small alphabets: one warp, no block barriers
    if (threadIdx.x < 32) book_warp(J, Sp, a, key, wgt, parent, nsym, p2, gh, span, cmin, L, book, lut_off);
    return;
  }
  // 2. leaves sorted by (count, symbol): stable_sort (huffman.hpp:74-77)
  if (nsym > 1) bitonic_sort(key, p2);
  // 3. two-queue merge, leaf queue preferred on ties (huffman.hpp:91-109)
  if (nsym > 1 && threadIdx.x == 0) {
    const uint32_t n = nsym, total = 2 * n - 1;
    for (uint32_t i = 0; i < n; ++i) {
      wgt[i] = key[i] >> 32;
      parent[i] = -1;
    }
    uint32_t size = n, lh = 0, mh = n;
    uint64_t wl = wgt[0];
    while (size < total) {
      uint32_t ab[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const bool leaf_ok = lh < n;
        const bool merged_ok = mh < size;
        if (leaf_ok && (!merged_ok || wl <= wgt[mh])) {
          ab[k] = lh++;
          wl = lh < n ? wgt[lh] : 0;
        } else {
          ab[k] = mh++;
        }
      }
      wgt[size] = wgt[ab[0]] + wgt[ab[1]];
      parent[size] = -1;
      parent[ab[0]] = static_cast<int32_t>(size);
      parent[ab[1]] = static_cast<int32_t>(size);
      ++size;
    }
  }
  if (threadIdx.x == 0) s_cap = ~0ull;
  __syncthreads();
  // 4. code lengths = leaf depth; the first leaf (sorted order) past 32 bits
  //    fails with its depth (huffman.hpp:110-118)
  for (uint32_t i = threadIdx.x; i < nsym; i += blockDim.x) {
    uint32_t depth = 0;
    if (nsym == 1) depth = 1;
    else
      for (int32_t p = parent[i]; p != -1; p = parent[p]) ++depth;
    if (depth > 32) atomicMin(&s_cap, (static_cast<unsigned long long>(i) << 32) | depth);
    const uint64_t sym = key[i] & 0xFFFFFFFFull;  // canonical key (length, symbol) (huffman.hpp:166-168)
    wgt[i] = (static_cast<uint64_t>(depth > 32 ? 63 : depth) << 32) | sym;
  }
  __syncthreads();
  if (s_cap != ~0ull) {
    if (threadIdx.x == 0) {
      Sp->aux = s_cap & 0xFFFFFFFFull;
      atomicMin(reinterpret_cast<unsigned long long*>(&Sp->err), err_key(s_cap >> 32, EMBC_R_HUF_LEN_CAP) | (1ull << 63));
      atomicOr(&a.flags[CF_ABORT], JF_ABORT);
    }
    for (uint64_t b = threadIdx.x; b < span; b += blockDim.x) gh[b] = 0;
    return;
  }
  // 5. canonical order (length asc, symbol asc)
  uint64_t* ckey = wgt;
  for (uint32_t i = nsym + threadIdx.x; i < p2; i += blockDim.x) ckey[i] = ~0ull;
  __syncthreads();
  if (nsym > 1) bitonic_sort(ckey, p2);
  // 6. canonical codes: code_i = sum_{j<i} 2^(len_i - len_j), the closed form
  //    of finalize's shift-and-increment (huffman.hpp:170-181)
  uint64_t bits_local = 0;
  {
    uint64_t carry = 0;
    for (uint32_t i0 = 0; i0 < nsym; i0 += blockDim.x) {
      const uint32_t i = i0 + threadIdx.x;
      uint32_t len = 0, symoff = 0;
      uint64_t kraft = 0;
      if (i < nsym) {
        len = static_cast<uint32_t>(ckey[i] >> 32);
        symoff = static_cast<uint32_t>(ckey[i]);
        kraft = 1ull << (32 - len);
      }
      unsigned long long tot;
      const unsigned long long pre = block_excl_scan<unsigned long long>(kraft, s_tmp64, &tot);
      if (i < nsym) {
        const uint64_t prefix = carry + pre;
        const uint32_t cw = static_cast<uint32_t>(prefix >> (32 - len));
        L[symoff] = (static_cast<uint64_t>(cw) << 8) | len;
        const int32_t sym = static_cast<int32_t>(static_cast<int64_t>(cmin) + symoff);
        uint8_t* e = book + 12 + 5ull * i;
        st_be(e, static_cast<uint32_t>(sym), 4);
        e[4] = static_cast<uint8_t>(len);
        bits_local += static_cast<uint64_t>(__ldcg(gh + symoff)) * len;
      }
      carry += tot;
    }
  }
  const unsigned long long bits = block_sum<unsigned long long>(bits_local, s_tmp64);
  for (uint64_t b = threadIdx.x; b < span; b += blockDim.x) gh[b] = 0;  // clean for the next call
  if (threadIdx.x == 0) {
    st_be(book, J.N, 8);       // u64be symbol_count (huffman.hpp:203)
    st_be(book + 8, nsym, 4);  // u32be entry_count (huffman.hpp:204)
    Sp->nsym = nsym;
    Sp->bits = bits;
    Sp->lut_off = lut_off;
    Sp->payload = 12 + 5ull * nsym + (bits + 7) / 8;
  }
}


// ---------------------------------------------------------------------------
// E1: quantize + per-tile statistics (+ codebook tail)
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// vlz matching of one tile (vlz.hpp:86-103): for every row the nearest
// earlier row inside the window with identical codes.  Candidates come from
// the row hashes nearest first and are verified exactly for all rows of the
// tile at once (CodeRowEq, vlz.hpp:75-79); a hash collision resumes the search
// past the disproved candidate.  `codes` holds the tile's codes (row r at
// r * stride); the window's hashes are read through L2 (other CTAs of the
// launch wrote them).  Writes row_dec; returns the tile's token bytes and
// counts reference rows in *nref.
// ---------------------------------------------------------------------------
struct VlzSmem {
  uint32_t* sh;       // staged window hashes (hash_cap)
  uint32_t* dec;      // per row: match offset (0 = literal)
  uint32_t* cand;     // per row: candidate offset under test
  uint32_t* plist;    // rows with a pending candidate
  uint32_t* miss;     // candidate disproved
  uint32_t* bhead;    // bucket chains over the staged hashes
  uint32_t chain_bytes;
  uint32_t hash_cap;
};

__device__ uint64_t vlz_match_tile(const DJob& J, const DTile& T, const int32_t* codes, uint32_t stride,
                                   const uint64_t* __restrict__ ri, uint32_t* __restrict__ row_dec, const VlzSmem& m,
                                   uint32_t* s_tmp32, unsigned long long* s_tmp64, uint64_t* nref_out) {
  const uint32_t dim = J.dim;
  const uint32_t W = J.window;
  const uint32_t lo = T.row0 > W ? T.row0 - W : 0;
  const uint32_t nh = T.row0 + T.rows - lo;
  const bool staged = nh <= m.hash_cap;
  uint32_t* sh = m.sh;
  uint32_t* dec = m.dec;
  uint32_t* cand = m.cand;
  uint32_t* plist = m.plist;
  uint32_t* miss = m.miss;
  if (staged)
    for (uint32_t k = threadIdx.x; k < nh; k += kBlock) sh[k] = static_cast<uint32_t>(__ldcg(ri + lo + k));
  // bucket chains (u16 links into sh): a row scans its 16 nearest offsets,
  // then walks its bucket for the nearest farther candidate
  uint32_t nbk = 0;
  if (staged && nh < 65535 && m.chain_bytes > 2 * nh + 4 * 256) {
    nbk = 4096;
    while (4 * nbk + 2 * nh > m.chain_bytes) nbk >>= 1;
    if (nbk < nh / 2) nbk = 0;
  }
  uint32_t* bhead = m.bhead;
  uint16_t* bnext = reinterpret_cast<uint16_t*>(bhead + nbk);
  const uint32_t bsh = 32 - (31 - __clz(nbk | 1));
  for (uint32_t k = threadIdx.x; k < nbk; k += kBlock) bhead[k] = 0xFFFFu;
  __syncthreads();
  for (uint32_t k = threadIdx.x; k < (nbk ? nh : 0); k += kBlock)
    bnext[k] = static_cast<uint16_t>(atomicExch(&bhead[(sh[k] * 0x9E3779B1u) >> bsh], k));
  __syncthreads();
  // nearest earlier row with an equal hash at offset >= k0, or 0
  auto search = [&](uint32_t r, uint32_t k0) -> uint32_t {
    const uint32_t i = T.row0 + r;
    const uint32_t kmax = min(W, i);
    if (!staged) {
      const uint32_t h = static_cast<uint32_t>(__ldcg(ri + i));
      for (uint32_t k = k0; k <= kmax; ++k)
        if (static_cast<uint32_t>(__ldcg(ri + i - k)) == h) return k;
      return 0;
    }
    const uint32_t h = sh[i - lo];
    const uint32_t knear = nbk ? min(kmax, k0 + 15) : kmax;
    uint32_t k = k0;
    for (; k + 3 <= knear; k += 4) {
      const uint32_t j = i - k - lo;
      const uint32_t h0 = sh[j], h1 = sh[j - 1], h2 = sh[j - 2], h3 = sh[j - 3];
      if (h0 == h) return k;
      if (h1 == h) return k + 1;
      if (h2 == h) return k + 2;
      if (h3 == h) return k + 3;
    }
    for (; k <= knear; ++k)
      if (sh[i - k - lo] == h) return k;
    if (knear >= kmax) return 0;
    // farther: the largest staged index e with i - kmax <= lo + e <= i - knear - 1
    const uint32_t ehi = i - knear - 1 - lo, elo = i - kmax - lo;
    uint32_t best = 0xFFFFFFFFu;
    for (uint32_t e = bhead[(h * 0x9E3779B1u) >> bsh]; e != 0xFFFFu; e = bnext[e])
      if (e <= ehi && e >= elo && sh[e] == h && (best == 0xFFFFFFFFu || e > best)) best = e;
    return best == 0xFFFFFFFFu ? 0 : i - lo - best;
  };
  for (uint32_t r = threadIdx.x; r < T.rows; r += kBlock) {
    cand[r] = search(r, 1);
    dec[r] = 0;
  }
  __syncthreads();
  const bool vq = (dim & 3) == 0 && stride == dim && (reinterpret_cast<uintptr_t>(J.src) & 15) == 0;
  for (;;) {
    uint32_t np = 0;  // compact the rows with a candidate under test
    for (uint32_t r0 = 0; r0 < T.rows; r0 += kBlock) {
      const uint32_t r = r0 + threadIdx.x;
      const bool p = r < T.rows && cand[r] != 0;
      uint32_t tot;
      const uint32_t at = block_excl_scan<uint32_t>(p, s_tmp32, &tot);
      if (p) {
        plist[np + at] = r;
        miss[np + at] = 0;
      }
      np += tot;
    }
    if (np == 0) break;
    __syncthreads();
    const uint32_t work = vq ? np * (dim >> 2) : np * dim;
    if (vq) {  // four codes per work item: 16-B smem / global loads
      const uint32_t qpr = dim >> 2;
      for (uint32_t e0w = 0; e0w < work; e0w += 2 * kBlock) {
        int4 cj[2], ci[2];
        uint32_t pp[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t e = e0w + u * kBlock + threadIdx.x;
          pp[u] = 0xFFFFFFFFu;
          if (e < work) {
            const uint32_t pi = e / qpr;
            const uint32_t qc = e - pi * qpr;
            const uint32_t r = plist[pi];
            const uint32_t i = T.row0 + r, j = i - cand[r];
            pp[u] = pi;
            ci[u] = reinterpret_cast<const int4*>(codes + r * dim)[qc];
            if (j >= T.row0) {
              cj[u] = reinterpret_cast<const int4*>(codes + (j - T.row0) * dim)[qc];
            } else {
              const uint4 g = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint32_t*>(J.src) +
                                                                   static_cast<uint64_t>(j) * dim) + qc);
              cj[u] = make_int4(static_cast<int32_t>(g.x), static_cast<int32_t>(g.y), static_cast<int32_t>(g.z),
                                static_cast<int32_t>(g.w));
              if (J.src_kind == EMBC_SRC_F32) pp[u] |= 0x80000000u;  // needs quantizing
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (pp[u] == 0xFFFFFFFFu) continue;
          int4 c = cj[u];
          if (pp[u] & 0x80000000u) {
            uint32_t rr = 0;
            c.x = quantize_f32(__int_as_float(c.x), J.qp, &rr);
            c.y = quantize_f32(__int_as_float(c.y), J.qp, &rr);
            c.z = quantize_f32(__int_as_float(c.z), J.qp, &rr);
            c.w = quantize_f32(__int_as_float(c.w), J.qp, &rr);
          }
          if (c.x != ci[u].x || c.y != ci[u].y || c.z != ci[u].z || c.w != ci[u].w) miss[pp[u] & 0x7FFFFFFFu] = 1;
        }
      }
    } else {
      for (uint32_t e0w = 0; e0w < work; e0w += 4 * kBlock) {
        int32_t cj[4], ci[4];
        uint32_t pp[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // all loads first: four rows' elements in flight
          const uint32_t e = e0w + u * kBlock + threadIdx.x;
          pp[u] = 0xFFFFFFFFu;
          if (e < work) {
            const uint32_t pi = fdiv(e, J.fd);
            const uint32_t col = e - pi * dim;
            const uint32_t r = plist[pi];
            const uint32_t i = T.row0 + r, j = i - cand[r];
            pp[u] = pi;
            ci[u] = codes[r * stride + col];
            if (j >= T.row0) {
              cj[u] = codes[(j - T.row0) * stride + col];
            } else if (J.src_kind == EMBC_SRC_F32) {
              cj[u] = __float_as_int(__ldg(static_cast<const float*>(J.src) + static_cast<uint64_t>(j) * dim + col));
              pp[u] |= 0x80000000u;  // needs quantizing
            } else {
              cj[u] = __ldg(static_cast<const int32_t*>(J.src) + static_cast<uint64_t>(j) * dim + col);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (pp[u] == 0xFFFFFFFFu) continue;
          int32_t c = cj[u];
          if (pp[u] & 0x80000000u) {
            uint32_t rr = 0;
            c = quantize_f32(__int_as_float(c), J.qp, &rr);
          }
          if (c != ci[u]) miss[pp[u] & 0x7FFFFFFFu] = 1;
        }
      }
    }
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < np; q += kBlock) {
      const uint32_t r = plist[q];
      if (!miss[q]) {
        dec[r] = cand[r];
        cand[r] = 0;
      } else {  // hash collision: keep looking further back
        cand[r] = search(r, cand[r] + 1);
      }
    }
    __syncthreads();
  }
  unsigned long long local = 0, nref = 0;
  for (uint32_t r = threadIdx.x; r < T.rows; r += kBlock) {
    const uint32_t found = dec[r];
    local += found ? 1u + varint_len(found) : static_cast<uint32_t>(__ldcg(ri + T.row0 + r) >> 32);
    nref += found != 0;
    row_dec[T.row0 + r] = found;
  }
  const unsigned long long both = block_sum<unsigned long long>(local | (nref << 40), s_tmp64);
  *nref_out = both >> 40;
  return both & ((1ull << 40) - 1);
}

struct StatsArgs {
  const DJob* jobs;
  const DTile* tiles;
  JobState* st;
  uint64_t* row_info;                 // vlz: (literal token bytes << 32) | row hash
  unsigned long long* tile_status;    // zeroed here for E2
  unsigned long long* job_status;
  uint32_t* edge_slot;
  BookArgs book;
  uint32_t hist_off;  // dynamic smem offset of the histogram window / vlz matching scratch
  // vlz matching (vlz.hpp:86-103) runs in E1: a tile publishes its row hashes,
  // waits for the tiles its window reaches into, then matches its rows
  uint32_t* row_dec;                  // per row: match offset (0 = literal)
  uint32_t* hready;                   // per tile: row hashes published (zeroed by the upload)
  unsigned long long* d_stats;        // match_stats: (literal rows, reference rows)
  uint32_t hash_cap, rows_cap, chain_bytes;
  uint32_t match;                     // match here (fused E2 / match_stats); else E2's sizes pass does
  // two-pass calls: a huffman tile's histogram (codes tile_hr.x .. + tile_hr.y),
  // so E2's sizes pass prices the tile without re-reading it (y == 0: re-read)
  uint32_t* tile_hist;
  int2* tile_hr;
};

// E1's vector loop, one instantiation per codec (no codec branches inside):
// 128-bit loads, 4 quads in flight per thread; a vlz row is qpr consecutive lanes.
template <int CODEC, bool STAGE_HUF>
__device__ __forceinline__ void stats_vec(const DJob& J, uint64_t e0, uint32_t ne, uint32_t qpr, uint64_t gbase,
                                          uint64_t* __restrict__ row_info, uint32_t* shist, int32_t* codes,
                                          unsigned long long& lerr, int& lmin, int& lmax, bool& lwide) {
  constexpr bool vlz = CODEC == EMBC_CODEC_VLZ, huf = CODEC == EMBC_CODEC_HUFFMAN;
  const uint32_t nq = ne >> 2;
  const QParams qp = J.qp;
  const bool f32 = J.src_kind == EMBC_SRC_F32;
  const uint4* src4 = reinterpret_cast<const uint4*>(static_cast<const uint32_t*>(J.src) + e0);
  uint32_t ck[4] = {0, 0, 0, 0};  // this thread's columns are fixed: q % qpr == threadIdx.x % qpr
  if (vlz)
#pragma unroll
    for (int k = 0; k < 4; ++k) ck[k] = col_key((threadIdx.x & (qpr - 1)) * 4 + k);
  for (uint32_t base = 0; base < nq; base += 4 * kBlock) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t q = base + u * kBlock + threadIdx.x;
      if (q < nq) v[u] = __ldg(src4 + q);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t q = base + u * kBlock + threadIdx.x;
      const bool ok = q < nq;
      int32_t c[4] = {0, 0, 0, 0};
      if (ok) {
        const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (f32) {
            uint32_t reason = 0;
            c[k] = quantize_f32(__uint_as_float(w[k]), qp, &reason);
            if (reason) lerr = min(lerr, static_cast<unsigned long long>(err_key(e0 + 4ull * q + k, reason)));
          } else {
            c[k] = static_cast<int32_t>(w[k]);
          }
          if (huf) {
            lmin = min(lmin, c[k]);
            lmax = max(lmax, c[k]);
            if (STAGE_HUF) {
              const uint32_t l = 4 * q + k;
              codes[l + (l >> 5)] = c[k];
            }
          }
        }
      }
      if (huf) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t bin = 0xFFFFFFFFu;
          if (ok) {
            const uint32_t b = static_cast<uint32_t>(c[k] + static_cast<int32_t>(kWin / 2));
            if (b < kWin) bin = b;
            else lwide = true;
          }
          hist_add(shist, bin);
        }
      }
      if (vlz) {
        uint32_t h = 0, lit = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          h += static_cast<uint32_t>(c[k]) * ck[k];
          lit += varint_len(zigzag(c[k]));
        }
        for (uint32_t o = 1; o < qpr; o <<= 1) {
          h += __shfl_xor_sync(0xffffffffu, h, o);
          lit += __shfl_xor_sync(0xffffffffu, lit, o);
        }
        if (ok && (q & (qpr - 1)) == 0) row_info[gbase + q / qpr] = (static_cast<uint64_t>(1 + lit) << 32) | h;
        if (ok) reinterpret_cast<int4*>(codes)[q] = make_int4(c[0], c[1], c[2], c[3]);  // row-major, for matching
      }
    }
  }
}

// E1 on one tile.  MERGED (the single-launch encode of small calls): the
// tile's codes stay in shared memory for E2 (huffman padded l + l/32, vlz
// row-major), the codebook scratch lives past them (smem + hist_off), and the
// job's codebook is published through JobState::flags.
template <bool MERGED>
__device__ __forceinline__ void stats_tile(const StatsArgs& a, const uint32_t tid, uint8_t* smem) {
  __shared__ unsigned long long s_err;
  __shared__ int s_min, s_max, s_last;
  TS1(0);
  const DTile T = a.tiles[tid];
  const DJob& J = a.jobs[T.job];
  if (threadIdx.x == 0) {
    s_err = ~0ull;
    s_min = INT_MAX;
    s_max = INT_MIN;
  }
  const uint32_t dim = J.dim;
  const bool vlz = J.codec == EMBC_CODEC_VLZ;
  const bool huf = J.codec == EMBC_CODEC_HUFFMAN;
  uint32_t* shist = reinterpret_cast<uint32_t*>(smem + a.hist_off);
  if (huf)
    for (uint32_t b = threadIdx.x; b < kWin; b += blockDim.x) shist[b] = 0;
  __syncthreads();

  const uint64_t e0 = static_cast<uint64_t>(T.row0) * dim;
  const uint32_t ne = T.rows * dim;
  unsigned long long lerr = ~0ull;
  int lmin = INT_MAX, lmax = INT_MIN;
  bool lwide = false;
  const uint32_t qpr = dim >> 2;  // quads per row
  const bool vec = (dim & 3) == 0 && (reinterpret_cast<uintptr_t>(J.src) & 15) == 0 &&
                   (!vlz || (qpr <= 32 && (qpr & (qpr - 1)) == 0));
  const uint64_t gbase = J.row_base + T.row0;
  if (vec) {
    int32_t* codes = reinterpret_cast<int32_t*>(smem);
    if (vlz) stats_vec<EMBC_CODEC_VLZ, false>(J, e0, ne, qpr, gbase, a.row_info, shist, codes, lerr, lmin, lmax, lwide);
    else if (huf)
      stats_vec<EMBC_CODEC_HUFFMAN, MERGED>(J, e0, ne, qpr, gbase, a.row_info, shist, codes, lerr, lmin, lmax, lwide);
    else stats_vec<EMBC_CODEC_RAW, false>(J, e0, ne, qpr, gbase, a.row_info, shist, codes, lerr, lmin, lmax, lwide);
  } else {
    // generic path: element loop, vlz codes staged at r * (dim|1) + col
    int32_t* codes = reinterpret_cast<int32_t*>(smem);
    const uint32_t stride = MERGED ? dim : (dim | 1u);  // MERGED: E2's row-major layout
    for (uint32_t l0 = 0; l0 < ne; l0 += kBlock) {
      const uint32_t l = l0 + threadIdx.x;
      const bool ok = l < ne;
      int32_t c = 0;
      if (ok) {
        uint32_t reason = 0;
        c = job_code(J, e0 + l, &reason);
        if (reason) lerr = min(lerr, static_cast<unsigned long long>(err_key(e0 + l, reason)));
        lmin = min(lmin, c);
        lmax = max(lmax, c);
      }
      if (huf) {
        uint32_t bin = 0xFFFFFFFFu;
        if (ok) {
          const uint32_t b = static_cast<uint32_t>(c + static_cast<int32_t>(kWin / 2));
          if (b < kWin) bin = b;
          else lwide = true;
        }
        hist_add(shist, bin);
      }
      if (vlz && ok) {
        const uint32_t r = fdiv(l, J.fd);
        codes[r * stride + (l - r * dim)] = c;
      }
      if (MERGED && huf && ok) codes[l + (l >> 5)] = c;
    }
    if (vlz) {
      __syncthreads();
      for (uint32_t r = threadIdx.x; r < T.rows; r += blockDim.x) {
        const int32_t* row = codes + r * stride;
        uint32_t h = 0, lit = 1;
        for (uint32_t j = 0; j < dim; ++j) {
          h += static_cast<uint32_t>(row[j]) * col_key(j);
          lit += varint_len(zigzag(row[j]));
        }
        a.row_info[gbase + r] = (static_cast<uint64_t>(lit) << 32) | h;
      }
    }
  }
  TS1(1);
  TS1(3);
  TS1(4);
  // fold the tile's failure key and code range into the job state
  JobState* Sp = &a.st[T.job];
  lerr = warp_min_u64(lerr);
  if ((threadIdx.x & 31) == 0 && lerr != ~0ull) atomicMin(&s_err, lerr);
  if (huf) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
      lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&s_min, lmin);
      atomicMax(&s_max, lmax);
    }
  }
  const bool wide = __syncthreads_or(lwide);
  if (threadIdx.x == 0) {
    if (s_err != ~0ull) {
      atomicMin(reinterpret_cast<unsigned long long*>(&Sp->err), s_err);
      atomicOr(&a.book.flags[CF_ABORT], JF_ABORT);
    }
    if (huf && ne) {
      atomicMin(&Sp->cmin, s_min);
      atomicMax(&Sp->cmax, s_max);
      if (wide) Sp->wide = 1;
    }
  }
  if (huf && !wide && ne) {  // flush the occupied bins of the window
    uint32_t* gh = a.book.hist + static_cast<uint64_t>(J.hjob) * kWin;
    const uint32_t b0 = static_cast<uint32_t>(s_min + static_cast<int32_t>(kWin / 2));
    const uint32_t b1 = static_cast<uint32_t>(s_max + static_cast<int32_t>(kWin / 2));
    const bool keep = !MERGED && a.tile_hist && b1 - b0 < kTileHist;
    for (uint32_t b = b0 + threadIdx.x; b <= b1; b += blockDim.x) {
      const uint32_t v = shist[b];
      if (v) atomicAdd(&gh[b], v);
      if (keep) a.tile_hist[static_cast<uint64_t>(tid) * kTileHist + (b - b0)] = v;
    }
    if (a.tile_hr && threadIdx.x == 0)  // a span past kTileHist is not kept: (0, 0) = re-read
      a.tile_hr[tid] = keep ? make_int2(s_min, static_cast<int>(b1 - b0 + 1)) : make_int2(0, 0);
  } else if (!MERGED && a.tile_hr && threadIdx.x == 0) {
    a.tile_hr[tid] = make_int2(0, 0);
  }
  TS1(2);
  if (vlz && a.match) {
    // publish this tile's row hashes, wait for the tiles the window reaches
    // into (earlier tickets of the same job), then match
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) *reinterpret_cast<volatile uint32_t*>(&a.hready[tid]) = 1;
    if (!J.window_ok || T.rows == 0) return;
    const uint32_t lo = T.row0 > J.window ? T.row0 - J.window : 0;
    for (uint32_t t = J.tile0 + lo / J.tile_rows + threadIdx.x; t < tid; t += blockDim.x) {
      uint32_t delay = 32;
      while (!*reinterpret_cast<volatile uint32_t*>(&a.hready[t])) {
        __nanosleep(delay);
        delay = min(delay * 2, kPollMaxNs);
      }
    }
    __threadfence();
    __syncthreads();
    __shared__ uint32_t s_tmp32[33];
    __shared__ unsigned long long s_tmp64[33];
    uint32_t* aux = reinterpret_cast<uint32_t*>(smem + a.hist_off);
    VlzSmem m;
    m.sh = aux;
    m.dec = aux + a.hash_cap;
    m.cand = m.dec + a.rows_cap;
    m.plist = m.cand + a.rows_cap;
    m.miss = m.plist + a.rows_cap;
    m.bhead = m.miss + a.rows_cap;
    m.chain_bytes = a.chain_bytes;
    m.hash_cap = a.hash_cap;
    uint64_t nref = 0;
    vlz_match_tile(J, T, reinterpret_cast<const int32_t*>(smem), vec || MERGED ? dim : (dim | 1u), a.row_info + J.row_base,
                   a.row_dec + J.row_base, m, s_tmp32, s_tmp64, &nref);
    if (a.d_stats && threadIdx.x == 0) {  // match_stats (vlz.hpp:162-168)
      atomicAdd(&a.d_stats[0], static_cast<unsigned long long>(T.rows) - nref);
      atomicAdd(&a.d_stats[1], static_cast<unsigned long long>(nref));
    }
    return;
  }
  if (!huf) return;
  // the job's last tile to finish builds the codebook
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&Sp->tiles_done, 1u) == J.ntiles - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  TS1(3);
  build_book(J, Sp, a.book, MERGED ? smem + a.hist_off : smem);
  if (MERGED) {  // the job's codebook (or its failure) is final
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      // the codebook prices the whole payload (count x length per symbol), so
      // the job's size is known here: publish it for the job look-back now
      // rather than after every tile of the job has sized itself in E2 (which
      // then finds it set).  Job 0 only ever publishes its inclusive offset.
      if (T.job > 0 && *reinterpret_cast<const volatile unsigned long long*>(&Sp->err) == ~0ull)
        atomicCAS(a.job_status + T.job * kJobStride, 0ull, kFlagAgg | (J.header + Sp->payload));
      *reinterpret_cast<volatile uint32_t*>(&Sp->flags) = 1;
    }
  }
  TS1(4);
}

__global__ void __launch_bounds__(kBlock, 4) k_stats(StatsArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  // tile = block index: a vlz tile only ever waits on lower tiles, which are
  // dispatched first (block-index order, as CUB's single-pass scans assume)
  stats_tile<false>(a, blockIdx.x, smem);
}

// ---------------------------------------------------------------------------
// E2: sizes -> decoupled look-back -> bytes
// ---------------------------------------------------------------------------
struct EmitArgs {
  const DJob* jobs;
  const DTile* tiles;
  JobState* st;
  const uint64_t* row_info;
  unsigned long long* tile_status;
  unsigned long long* job_status;
  uint32_t* edge_slot;
  const uint64_t* lut;
  const uint8_t* books;
  uint64_t book_stride;
  uint32_t* flags;
  uint32_t njobs, ntiles;
  int layout;
  uint8_t* out;
  uint64_t cap;
  uint64_t* d_offsets;
  uint64_t* d_lengths;
  uint8_t* d_meta;
  uint64_t* d_total;
  DevError* err;
  unsigned long long* d_stats;  // match_stats mode: (literals, references); no bytes
  uint32_t stage_off, aux_off;  // dynamic smem carve
  uint32_t hash_cap, rows_cap;  // aux: staged row hashes | 5 per-row arrays
  uint32_t* row_dec;            // vlz: match offset per row (phase 0 -> phase 1)
  uint64_t* tile_bits;          // payload bits per tile (phase 0)
  uint64_t* tile_off;           // bit offset of each tile inside its job's payload data (layout)
  uint64_t* job_start;          // chunk offset of each job (layout)
  uint32_t* done;               // phase-0 completion ticket
  int phase;                    // 0: sizes + layout (last CTA), 1: bytes
  const uint32_t* tile_hist;    // huffman tiles priced from E1's histograms (phase 0)
  const int2* tile_hr;
};

__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// Warp-cooperative decoupled look-back: the exclusive prefix of element `i`
// over status[first .. i-1], where status[first] always publishes an
// inclusive value and `base` is the prefix before `first`.

__device__ __forceinline__ uint64_t look_back(const unsigned long long* status, uint32_t first, uint32_t i,
                                              uint64_t base, uint32_t stride = 1) {
  const uint32_t lane = threadIdx.x & 31;
  uint64_t acc = 0;
  int64_t p = static_cast<int64_t>(i) - 1;
  uint32_t delay = 32;
  while (p >= static_cast<int64_t>(first)) {
    const int64_t idx = p - lane;
    unsigned long long s = kFlagInc;  // before `first`: inclusive 0 (never reached: first is inclusive)
    if (idx >= static_cast<int64_t>(first)) s = ld_status(status + idx * stride);
    const uint32_t inc = __ballot_sync(0xffffffffu, (s >> 62) == 2);
    const uint32_t zero = __ballot_sync(0xffffffffu, (s >> 62) == 0);
    const int fi = inc ? __ffs(inc) - 1 : 32;
    const uint32_t need = fi == 32 ? 0xffffffffu : ((2u << fi) - 1);
    if (zero & need) {  // a predecessor has not published yet: back off, re-read
      EMBC_DBG(if (lane == 0) atomicAdd(&g_dbg[stride == 1 ? 0 : 1], 1ull));
      __nanosleep(delay);
      delay = min(delay * 2, kPollMaxNs);
      continue;
    }
    uint64_t v = (static_cast<int>(lane) <= fi) ? (s & kValMask) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    acc += v;
    if (fi < 32) return acc;
    p -= 32;
  }
  return acc + base;
}

// Look-back status words carry their value (tile bits, job offsets) and
// publish no other data: a volatile store, no fence.
__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
  *reinterpret_cast<volatile unsigned long long*>(p) = v;
}

// fold the lowest failing job into the sticky record (layout order)
__device__ void fold_failure(const EmitArgs& a) {
  __shared__ unsigned long long s_first;
  if (threadIdx.x == 0) s_first = ~0ull;
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < a.njobs; j += blockDim.x)
    if (a.st[j].err != ~0ull) atomicMin(&s_first, static_cast<unsigned long long>(j));
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (a.d_total) *a.d_total = 0;
  if (s_first == ~0ull || a.err->valid) return;
  const uint32_t j = static_cast<uint32_t>(s_first);
  const unsigned long long k = a.st[j].err & ~(1ull << 63);
  a.err->valid = 1;
  a.err->job = j;
  a.err->reason = static_cast<int32_t>(k & 63);
  a.err->index = k >> 6;
  a.err->a = a.st[j].aux;
  a.err->b = a.jobs[j].window;
  a.err->eb = a.jobs[j].qp.eb;
  a.err->status = (a.err->reason == EMBC_R_RANGE) ? EMBC_ERR_UNSUPPORTED : EMBC_ERR_VALUE;
}

// copy [a, b) of the staged bytes (stage[mis + k] <-> dst[k]) with 16-B stores
__device__ __forceinline__ void copy_range(uint8_t* dst, const uint8_t* stage, uint32_t mis, uint64_t a, uint64_t b) {
  if (b <= a) return;
  const uint32_t m2 = (mis + static_cast<uint32_t>(a)) & 15u;
  copy_out_staged(dst + a, stage + (mis + a - m2), b - a);
}

// One chunk's records: pack table entry (container.hpp:244-250), header
// (container.hpp:74-85), 25-B metadata (container.hpp:196-209), offsets.
__device__ void write_job_records(const EmitArgs& a, uint32_t j, uint64_t start, uint64_t P) {
  const DJob& J = a.jobs[j];
  const uint64_t len = J.header + P;
  if (a.d_offsets) a.d_offsets[j] = start;
  if (a.d_lengths) a.d_lengths[j] = len;
  if (a.layout == EMBC_LAYOUT_PACKED && 20 + 16ull * j <= a.cap) {
    st_le(a.out + 4 + 16ull * j, start, 8);
    st_le(a.out + 12 + 16ull * j, len, 8);
  }
  uint64_t ebits;
  memcpy(&ebits, &J.qp.eb, 8);
  if (J.header && start + kHeader <= a.cap) {
    uint8_t* h = a.out + start;
    h[0] = 'E';
    h[1] = 'M';
    h[2] = 'B';
    h[3] = 'C';
    h[4] = 1;
    h[5] = J.codec;
    st_le(h + 6, ebits, 8);
    st_le(h + 14, J.dim, 4);
    st_le(h + 18, J.n, 4);
    st_le(h + 22, P, 8);
  }
  if (a.d_meta) {
    uint8_t* m = a.d_meta + static_cast<uint64_t>(kMetaSize) * j;
    st_le(m, kHeader + P, 8);
    m[8] = J.codec;
    st_le(m + 9, ebits, 8);
    st_le(m + 17, J.dim, 4);
    st_le(m + 21, J.n, 4);
  }
}

// The call's total: d_total, or the capacity error (then nothing more is written).
__device__ void finish_call(const EmitArgs& a, uint64_t total) {
  if (total > a.cap) {
    if (a.d_total) *a.d_total = 0;
    a.flags[CF_ABORT] |= JF_ABORT;
    if (!a.err->valid) {
      a.err->valid = 1;
      a.err->job = 0;
      a.err->reason = EMBC_R_CAPACITY;
      a.err->index = 0;
      a.err->a = total;
      a.err->b = a.cap;
      a.err->status = EMBC_ERR_CAPACITY;
    }
  } else if (a.d_total) {
    *a.d_total = total;
  }
}

// Layout of the call (the last phase-0 CTA): tile offsets inside each job's
// payload (bits), chunk offsets in job order (container.hpp:245-250), chunk
// headers (container.hpp:74-85), pack table (container.hpp:244-250), 25-B
// metadata (container.hpp:196-209), capacity check.
// Segmented scan operator over (segment started, value): a later element that
// starts a segment discards the running sum.
struct SegVal {
  unsigned long long v;
  uint32_t head;
};
__device__ __forceinline__ SegVal seg_op(SegVal a, SegVal b) {
  return SegVal{b.head ? b.v : a.v + b.v, a.head | b.head};
}

__device__ void layout_tail(const EmitArgs& a) {
  __shared__ unsigned long long s_tmp64[33];
  __shared__ unsigned long long s_wv[32];
  __shared__ uint32_t s_wh[32];
  __shared__ unsigned long long s_cv;
  // 1. every tile's bit offset inside its job's payload data: a segmented
  //    exclusive scan of the tile bits (segments = jobs, contiguous in tile
  //    order), kLT tiles per thread per round with all loads in flight; the
  //    job totals (last tile of each job) go straight to job_start
  constexpr uint32_t kLT = 8;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_cv = 0;
  __syncthreads();
  for (uint32_t r0 = 0; r0 < a.ntiles; r0 += kLT * blockDim.x) {
    const uint32_t t0 = r0 + threadIdx.x * kLT;
    unsigned long long bits[kLT];
    uint32_t job[kLT];
#pragma unroll
    for (uint32_t k = 0; k < kLT; ++k) {
      const uint32_t t = t0 + k;
      bits[k] = t < a.ntiles ? __ldcg(a.tile_bits + t) : 0;
      job[k] = t < a.ntiles ? a.tiles[t].job : 0xFFFFFFFFu;
    }
    // the job of the tile before this thread's first (segment head test)
    const uint32_t prevj = t0 == 0 ? 0xFFFFFFFEu : (t0 - 1 < a.ntiles ? a.tiles[t0 - 1].job : 0xFFFFFFFFu);
    // thread aggregate
    SegVal agg{0, 0};
    uint32_t pj = prevj;
#pragma unroll
    for (uint32_t k = 0; k < kLT; ++k) {
      const SegVal e{bits[k], job[k] != pj ? 1u : 0u};
      agg = seg_op(agg, e);
      pj = job[k];
    }
    // block-wide exclusive scan of the aggregates (warp shuffles, then warps)
    SegVal inc = agg;
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xffffffffu, inc.v, o);
      const uint32_t h = __shfl_up_sync(0xffffffffu, inc.head, o);
      if (lane >= o) inc = seg_op(SegVal{v, h}, inc);
    }
    if (lane == 31) {
      s_wv[warp] = inc.v;
      s_wh[warp] = inc.head;
    }
    __syncthreads();
    // exclusive prefix of this warp: the carry-in of the round, then earlier warps
    SegVal wpre{s_cv, 0};
    for (uint32_t w = 0; w < warp; ++w) wpre = seg_op(wpre, SegVal{s_wv[w], s_wh[w]});
    const unsigned long long xv = __shfl_up_sync(0xffffffffu, inc.v, 1);
    const uint32_t xh = __shfl_up_sync(0xffffffffu, inc.head, 1);
    const SegVal ex = lane ? seg_op(wpre, SegVal{xv, xh}) : wpre;
    // the tiles' offsets (and each job's total at its last tile)
    unsigned long long run = ex.v;
    pj = prevj;
#pragma unroll
    for (uint32_t k = 0; k < kLT; ++k) {
      const uint32_t t = t0 + k;
      if (t >= a.ntiles) break;
      if (job[k] != pj) run = 0;
      a.tile_off[t] = run;
      run += bits[k];
      pj = job[k];
      if (t + 1 == a.ntiles || (k + 1 < kLT ? job[k + 1] != job[k] : a.tiles[t + 1].job != job[k]))
        a.job_start[job[k]] = run;  // the job's payload bits (step 3 turns it into the chunk offset)
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_cv = seg_op(ex, agg).v;  // the round's carry-out
    __syncthreads();
  }
  __threadfence_block();
  __syncthreads();
  // 3. chunk sizes -> offsets in job order, then the per-chunk records
  const uint64_t base = a.layout == EMBC_LAYOUT_PACKED ? 4 + 16ull * a.njobs : 0;
  unsigned long long carry = base;
  for (uint32_t j0 = 0; j0 < a.njobs; j0 += blockDim.x) {
    const uint32_t j = j0 + threadIdx.x;
    uint64_t P = 0, len = 0;
    if (j < a.njobs) {
      const DJob& J = a.jobs[j];
      const uint64_t bits = __ldcg(a.job_start + j);  // the job's payload bits (step 1)
      P = (J.codec == EMBC_CODEC_HUFFMAN ? 12 + 5ull * a.st[j].nsym : 0) + (bits + 7) / 8;
      len = J.header + P;
    }
    unsigned long long tot;
    const unsigned long long pre = block_excl_scan<unsigned long long>(len, s_tmp64, &tot);
    if (j < a.njobs) {
      const DJob& J = a.jobs[j];
      const uint64_t start = carry + pre;
      a.job_start[j] = start;
      if (a.d_offsets) a.d_offsets[j] = start;
      if (a.d_lengths) a.d_lengths[j] = len;
      if (a.layout == EMBC_LAYOUT_PACKED && 20 + 16ull * j <= a.cap) {
        st_le(a.out + 4 + 16ull * j, start, 8);
        st_le(a.out + 12 + 16ull * j, len, 8);
      }
      uint64_t ebits;
      memcpy(&ebits, &J.qp.eb, 8);
      if (J.header && start + kHeader <= a.cap) {
        uint8_t* h = a.out + start;
        h[0] = 'E';
        h[1] = 'M';
        h[2] = 'B';
        h[3] = 'C';
        h[4] = 1;
        h[5] = J.codec;
        st_le(h + 6, ebits, 8);
        st_le(h + 14, J.dim, 4);
        st_le(h + 18, J.n, 4);
        st_le(h + 22, P, 8);
      }
      if (a.d_meta) {
        uint8_t* m = a.d_meta + static_cast<uint64_t>(kMetaSize) * j;
        st_le(m, kHeader + P, 8);
        m[8] = J.codec;
        st_le(m + 9, ebits, 8);
        st_le(m + 17, J.dim, 4);
        st_le(m + 21, J.n, 4);
      }
    }
    carry += tot;
  }
  if (threadIdx.x == 0) {
    const uint64_t total = carry;
    if (a.layout == EMBC_LAYOUT_PACKED && a.cap >= 4) st_le(a.out, a.njobs, 4);
    if (total > a.cap) {
      if (a.d_total) *a.d_total = 0;
      a.flags[CF_ABORT] |= JF_ABORT;  // phase 1 writes nothing
      if (!a.err->valid) {
        a.err->valid = 1;
        a.err->job = 0;
        a.err->reason = EMBC_R_CAPACITY;
        a.err->index = 0;
        a.err->a = total;
        a.err->b = a.cap;
        a.err->status = EMBC_ERR_CAPACITY;
      }
    } else if (a.d_total) {
      *a.d_total = total;
    }
  }
}

// E2 on one tile.  PHASE 0: sizes + layout (last CTA); 1: bytes; 2: fused
// (sizes, look-back, bytes).  MERGED (phase 2 after E1 in the same CTA): the
// codes are already in shared memory; the quantization verdict is final only
// once the look-back has passed, so a failed call still publishes every
// size (nothing ever waits forever), skips the bytes, and the last ticket folds
// the failure.
template <int PHASE, bool MERGED>
__device__ __forceinline__ void emit_tile(const EmitArgs& a, const uint32_t tid, uint8_t* smem) {
  __shared__ uint32_t s_tmp32[33];
  __shared__ unsigned long long s_tmp64[33];
  __shared__ unsigned long long s_pre, s_start, s_total;
  TS(0);
  EMBC_DBG(EmitEnd dbg_end{tid, PHASE == 2 ? a.ntiles : 0xFFFFFFFFu});
  if (!MERGED && (*reinterpret_cast<volatile uint32_t*>(&a.flags[CF_ABORT]) & JF_ABORT)) {
    if (tid == 0 && PHASE != 1 && !a.d_stats) fold_failure(a);
    return;
  }
  constexpr int phase = PHASE;
  const DTile T = a.tiles[tid];
  const uint32_t jid = T.job;
  const DJob J = a.jobs[jid];  // by value: the fields live in registers, not re-read after global stores
  const JobState& S = a.st[jid];
  const uint32_t dim = J.dim;
  const uint64_t e0 = static_cast<uint64_t>(T.row0) * dim;
  const uint32_t ne = T.rows * dim;
  const bool first = tid == J.tile0, last = tid == J.tile0 + J.ntiles - 1;
  int32_t* codes = reinterpret_cast<int32_t*>(smem);
  uint8_t* stage = smem + a.stage_off;
  uint8_t* aux = smem + a.aux_off;
  const uint32_t codec = J.codec;
  const uint32_t stride = codec == EMBC_CODEC_VLZ ? dim : 0;  // vlz rows unpadded: warps read rows along lanes
  EMBC_DBG(if (threadIdx.x == 0 && tid < 16384) g_tc[tid] = codec);

  uint32_t* dec = reinterpret_cast<uint32_t*>(aux + a.hash_cap * 4);  // vlz: match offset per row
  uint32_t* lits = dec + a.rows_cap;                                   // vlz: token bytes per row
  // vlz rows are matched in E1 (fused calls) or in phase 0: the byte passes
  // need the literal rows only
  const bool vlz_lit_only = codec == EMBC_CODEC_VLZ && phase != 0;
  if (vlz_lit_only) {
    const uint64_t* ri = a.row_info + J.row_base + T.row0;
    for (uint32_t r = threadIdx.x; r < T.rows; r += kBlock) {
      const uint32_t o = a.row_dec[J.row_base + T.row0 + r];
      dec[r] = o;
      lits[r] = o ? 1u + varint_len(o) : static_cast<uint32_t>((MERGED ? __ldcg(ri + r) : __ldg(ri + r)) >> 32);
    }
    __syncthreads();
  }
  // phase 0 prices a huffman tile from its E1 histogram when it was kept
  const int2 thr = (PHASE == 0 && codec == EMBC_CODEC_HUFFMAN && a.tile_hr) ? a.tile_hr[tid] : make_int2(0, 0);
  // ---- 1. codes of the tile into shared memory (vlz: row stride dim|1;
  //         huffman: l + l/32, conflict-free thread-contiguous reads)
  if (!MERGED && codec != EMBC_CODEC_RAW && ne && thr.y == 0) {
    const bool vec = (dim & 3) == 0 && (reinterpret_cast<uintptr_t>(J.src) & 15) == 0;
    if (vec) {
      const uint4* src4 = reinterpret_cast<const uint4*>(static_cast<const uint32_t*>(J.src) + e0);
      const uint32_t nq = ne >> 2;
      const bool f32 = J.src_kind == EMBC_SRC_F32;
      for (uint32_t base = 0; base < nq; base += 4 * kBlock) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t q = base + u * kBlock + threadIdx.x;
          if (q < nq && !(vlz_lit_only && dec[fdiv(4 * q, J.fd)])) v[u] = __ldg(src4 + q);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t q = base + u * kBlock + threadIdx.x;
          if (q >= nq || (vlz_lit_only && dec[fdiv(4 * q, J.fd)])) continue;
          const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
          int32_t vq[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t l = 4 * q + k;
            int32_t c;
            if (f32) {
              uint32_t r = 0;
              c = quantize_f32(__uint_as_float(w[k]), J.qp, &r);
            } else {
              c = static_cast<int32_t>(w[k]);
            }
            if (!stride) codes[l + (l >> 5)] = c;
            else vq[k] = c;
          }
          if (stride) reinterpret_cast<int4*>(codes)[q] = make_int4(vq[0], vq[1], vq[2], vq[3]);  // row-major
        }
      }
    } else {
      for (uint32_t l = threadIdx.x; l < ne; l += kBlock) {
        uint32_t at;
        uint32_t rr = 0;
        if (stride) {
          rr = fdiv(l, J.fd);
          at = rr * stride + (l - rr * dim);
          if (vlz_lit_only && dec[rr]) continue;
        } else {
          at = l + (l >> 5);
        }
        uint32_t r = 0;
        codes[at] = job_code(J, e0 + l, &r);
      }
    }
  }

  __syncthreads();
  TS(1);
  // ---- 2. tile size in bits (payload only; the header / codebook bytes are
  //         added at the job level)
  uint64_t my_bits = 0;
  uint32_t pos_thread = 0;                                              // huffman: this thread's first bit
  const uint32_t per_h = (ne + kBlock - 1) / kBlock;
  const uint64_t* L = a.lut + S.lut_off;
  uint64_t* sl = reinterpret_cast<uint64_t*>(aux);
  const int32_t cmin = S.cmin;
  const uint32_t span = codec == EMBC_CODEC_HUFFMAN ? static_cast<uint32_t>(S.cmax - cmin + 1) : 0;
  const bool lut_staged = span <= kLutStage && 8 * span <= a.hash_cap * 4 + a.rows_cap * 8;
  // MERGED: the LUT was written in this launch (L2 reads); a failed job has none
  auto ldL = [&](uint32_t k) -> uint64_t { return MERGED ? __ldcg(L + k) : __ldg(L + k); };
  const bool no_book = MERGED && codec == EMBC_CODEC_HUFFMAN &&
                       *reinterpret_cast<const volatile unsigned long long*>(&S.err) != ~0ull;
  if (codec == EMBC_CODEC_RAW) {
    my_bits = 32ull * ne;
  } else if (codec == EMBC_CODEC_VLZ && phase != 0) {  // matched before
    uint64_t local = 0;
    for (uint32_t r = threadIdx.x; r < T.rows; r += kBlock) local += lits[r];
    my_bits = 8ull * block_sum<unsigned long long>(local, s_tmp64);
  } else if (codec == EMBC_CODEC_VLZ) {  // phase 0 of a large call: match here
    VlzSmem m;
    m.sh = reinterpret_cast<uint32_t*>(aux);
    m.dec = dec;
    m.cand = lits + a.rows_cap;
    m.plist = m.cand + a.rows_cap;
    m.miss = m.plist + a.rows_cap;
    m.bhead = reinterpret_cast<uint32_t*>(stage);  // the output stage idles until the bytes pass
    m.chain_bytes = a.aux_off - a.stage_off;
    m.hash_cap = a.hash_cap;
    uint64_t nref = 0;
    my_bits = 8ull * vlz_match_tile(J, T, codes, stride, a.row_info + J.row_base, a.row_dec + J.row_base, m, s_tmp32,
                                    s_tmp64, &nref);
  } else if (no_book) {  // MERGED, quantization failed: sized empty, never emitted
    my_bits = 0;
  } else if (thr.y > 0) {  // phase 0: sum over the tile's histogram of count * code length
    uint64_t nb = 0;
    for (uint32_t b = threadIdx.x; b < static_cast<uint32_t>(thr.y); b += kBlock) {
      const uint32_t cnt = a.tile_hist[static_cast<uint64_t>(tid) * kTileHist + b];
      if (cnt) nb += static_cast<uint64_t>(cnt) * (ldL(static_cast<uint32_t>(thr.x + static_cast<int32_t>(b) - cmin)) & 0xFF);
    }
    my_bits = block_sum<unsigned long long>(nb, s_tmp64);
  } else {  // huffman
    if (lut_staged)
      for (uint32_t k = threadIdx.x; k < span; k += kBlock) sl[k] = ldL(k);
    __syncthreads();
    const uint32_t l0 = threadIdx.x * per_h, l1 = min(l0 + per_h, ne);
    uint32_t nb = 0;
    for (uint32_t l = l0; l < l1; ++l) {
      const uint32_t s = static_cast<uint32_t>(codes[l + (l >> 5)] - cmin);
      nb += static_cast<uint32_t>((lut_staged ? sl[s] : ldL(s)) & 0xFF);
    }
    uint32_t tot;
    pos_thread = block_excl_scan<uint32_t>(nb, s_tmp32, &tot);
    my_bits = tot;
  }

  TS(2);
  const uint64_t hdr = J.header;
  const uint64_t book_bytes = codec == EMBC_CODEC_HUFFMAN ? 12 + 5ull * S.nsym : 0;
  uint64_t pre = 0, start = 0;
  // phase 2: vlz / huffman tiles stage their bytes (from stage byte 0) before the job look-back
  constexpr bool prestage = PHASE == 2;
  uint32_t pst = 0;
  // vlz token stream (vlz.hpp:111-125) of the tile into stage + mis; returns its bytes
  auto stage_vlz = [&](uint32_t mis) -> uint32_t {
    uint32_t* roff = lits;  // token sizes -> byte offsets inside the tile (in place)
    const uint32_t per = (T.rows + kBlock - 1) / kBlock;
    const uint32_t r0 = threadIdx.x * per, r1 = min(r0 + per, T.rows);
    uint32_t sum = 0;
    for (uint32_t r = r0; r < r1; ++r) sum += lits[r];
    __syncthreads();
    uint32_t tot;
    uint32_t q0 = block_excl_scan<uint32_t>(sum, s_tmp32, &tot);
    for (uint32_t r = r0; r < r1; ++r) {
      const uint32_t sz = roff[r];
      roff[r] = q0;
      const uint32_t o = dec[r];
      if (o) {  // reference token: 0x01, varint(offset)
        uint8_t* q = stage + mis + q0;
        *q++ = 0x01;
        put_varint(q, o);
      }
      q0 += sz;
    }
    __syncthreads();
    // literal tokens: 0x00 then dim zigzag varints, one warp per row
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t r = warp; r < T.rows; r += kBlock / 32) {
      if (dec[r]) continue;
      uint8_t* q = stage + mis + roff[r];
      if (lane == 0) q[0] = 0x00;
      uint32_t carry = 1;
      const int32_t* row = codes + r * stride;
      for (uint32_t j0 = 0; j0 < dim; j0 += 32) {
        const uint32_t j = j0 + lane;
        uint32_t z = 0, len = 0;
        if (j < dim) {
          z = zigzag(row[j]);
          len = varint_len(z);
        }
        const uint32_t inc = warp_incl_scan<uint32_t>(len);
        if (j < dim) put_varint(q + carry + inc - len, z);
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    __syncthreads();
    return tot;
  };
  // huffman bitstream (bitstream.hpp:32-51) of the tile, MSB-first, into
  // stage from bit 8 * mis + (pre & 7); returns the staged bytes
  auto stage_huff = [&](uint32_t mis) -> uint32_t {
    uint32_t* words = reinterpret_cast<uint32_t*>(stage);
    const uint32_t lead = 8 * mis + static_cast<uint32_t>(pre & 7);
    const uint32_t endbit = lead + static_cast<uint32_t>(my_bits);
    const uint32_t nwords = (endbit + 31) / 32;
    for (uint32_t w = threadIdx.x; w < nwords + 1; w += kBlock) words[w] = 0;
    __syncthreads();
    {  // this thread's codes, assembled in a register and stored word by word
      const uint32_t l0 = threadIdx.x * per_h, l1 = min(l0 + per_h, ne);
      uint32_t q = lead + pos_thread;
      uint32_t wi = q >> 5, used = q & 31;
      uint64_t buf = 0;
      bool shared_word = true;  // the first word may be shared with the previous thread
      for (uint32_t l = l0; l < l1; ++l) {
        const uint32_t sy = static_cast<uint32_t>(codes[l + (l >> 5)] - cmin);
        const uint64_t e = lut_staged ? sl[sy] : ldL(sy);
        const uint32_t len = static_cast<uint32_t>(e & 0xFF);
        buf |= (e >> 8) << (64 - used - len);
        used += len;
        if (used >= 32) {
          const uint32_t w = static_cast<uint32_t>(buf >> 32);
          if (shared_word) atomicOr(&words[wi], w);
          else words[wi] = w;
          shared_word = false;
          buf <<= 32;
          used -= 32;
          ++wi;
        }
      }
      if (used) atomicOr(&words[wi], static_cast<uint32_t>(buf >> 32));  // may be shared with the next thread
    }
    __syncthreads();
    const uint32_t nbytes_stage = (endbit + 7) / 8;
    for (uint32_t w = threadIdx.x; w < (nbytes_stage + 3) / 4; w += kBlock) words[w] = __byte_perm(words[w], 0, 0x0123);
    __syncthreads();
    return nbytes_stage;
  };
  if (phase == 2) {
    // ---- 3c. fused: decoupled look-back over the job's tiles (bits), then over jobs (bytes)
    if (threadIdx.x == 0 && jid > 0) {
      // the job's size is known once every tile of it is sized: the last one to
      // get here publishes it, so later jobs never wait on this job's look-back
      unsigned long long* js = a.job_status + jid * kJobStride;
      atomicAdd(js + 1, static_cast<unsigned long long>(my_bits));
      __threadfence();
      if (atomicAdd(js + 2, 1ull) == J.ntiles - 1) {
        __threadfence();
        const unsigned long long bits = atomicAdd(js + 1, 0ull);
        const unsigned long long w = *reinterpret_cast<volatile unsigned long long*>(js);
        if ((w >> 62) == 0) atomicCAS(js, 0ull, kFlagAgg | (hdr + book_bytes + (bits + 7) / 8));
      }
    }

    uint64_t p = 0;
    if (threadIdx.x < 32) {
      if (first) {
        if (threadIdx.x == 0) st_status(a.tile_status + tid, kFlagInc | my_bits);
      } else {
        if (threadIdx.x == 0) st_status(a.tile_status + tid, kFlagAgg | my_bits);
        p = look_back(a.tile_status, J.tile0, tid, 0);
        if (threadIdx.x == 0) st_status(a.tile_status + tid, kFlagInc | (p + my_bits));
      }
      if (threadIdx.x == 0) s_pre = p;
    }
    if constexpr (prestage) {
      // the tile's bytes need only its bit offset inside the job: stage them
      // now (from stage byte 0) while the job look-back may still wait on an
      // earlier job's codebook; after it only the copy out remains
      if (codec != EMBC_CODEC_RAW && !no_book) {
        __syncthreads();
        pre = s_pre;
        pst = codec == EMBC_CODEC_VLZ ? stage_vlz(0) : stage_huff(0);
      }
    }
    if (threadIdx.x < 32) {
      const uint64_t job_bytes = hdr + book_bytes + (p + my_bits + 7) / 8;
      const uint64_t base = a.layout == EMBC_LAYOUT_PACKED ? 4 + 16ull * a.njobs : 0;
      const uint64_t st0 = jid == 0 ? base : look_back(a.job_status, 0, jid, 0, kJobStride);
      if (last && threadIdx.x == 0) st_status(a.job_status + jid * kJobStride, kFlagInc | (st0 + job_bytes));
      if (threadIdx.x == 0) {
        s_pre = p;
        s_start = st0;
      }
    }
    __syncthreads();
    TS(3);
    pre = s_pre;
    start = s_start;
    if (last && threadIdx.x == 0) {  // the job's records (header, pack table, metadata)
      const uint64_t P = book_bytes + (pre + my_bits + 7) / 8;
      write_job_records(a, jid, start, P);
      if (tid == a.ntiles - 1) {
        if (!MERGED) finish_call(a, start + hdr + P);
        else s_total = start + hdr + P;
      }
    }
    if (tid == 0 && threadIdx.x == 0 && a.layout == EMBC_LAYOUT_PACKED && a.cap >= 4) st_le(a.out, a.njobs, 4);
    if (MERGED) {
      // the last ticket is past every other tile's E1: the abort flag is final
      // there (earlier tiles may still emit bytes of a call that then fails)
      __shared__ int s_abort;
      __syncthreads();
      if (threadIdx.x == 0) s_abort = (*reinterpret_cast<volatile uint32_t*>(&a.flags[CF_ABORT]) & JF_ABORT) != 0;
      __syncthreads();
      if (tid == a.ntiles - 1) {
        if (s_abort) fold_failure(a);
        else if (threadIdx.x == 0) finish_call(a, s_total);
      }
      if (s_abort) return;
    }
  } else if (phase == 0) {
    // ---- 3a. sizes out; the last CTA to finish lays the call out
    __shared__ int s_last;
    if (threadIdx.x == 0) a.tile_bits[tid] = my_bits;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(a.done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    layout_tail(a);
    return;
  }
  if (phase == 1) {  // ---- 3b. offsets from the layout
    if (*reinterpret_cast<volatile uint32_t*>(&a.flags[CF_ABORT]) & JF_ABORT) return;  // capacity
    pre = a.tile_off[tid];
    start = a.job_start[jid];
  }
  const uint64_t pay_end = start + hdr + book_bytes + (pre + my_bits + 7) / 8;  // end of this tile's bytes
  uint8_t* pay = a.out + start + hdr;
  EMBC_DBG(dbg_stats_report(a));
  const bool fits = pay_end <= a.cap;

  // ---- 5. bytes
  if (codec == EMBC_CODEC_RAW) {  // u32le codes (container.hpp:128-133)
    if (!fits || !ne) return;
    uint8_t* dst = pay + 4 * e0;
    const uint32_t mis = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(dst) & 15);
    const bool vec = (dim & 3) == 0 && (reinterpret_cast<uintptr_t>(J.src) & 15) == 0 && J.src_kind == EMBC_SRC_F32;
    if (vec && mis == 0) {  // aligned: quantize straight into 16-B stores
      const uint4* src4 = reinterpret_cast<const uint4*>(static_cast<const float*>(J.src) + e0);
      uint4* d4 = reinterpret_cast<uint4*>(dst);
      for (uint32_t q = threadIdx.x; q < ne / 4; q += kBlock) {
        const uint4 v = __ldg(src4 + q);
        uint32_t r = 0;
        uint4 o;
        o.x = static_cast<uint32_t>(quantize_f32(__uint_as_float(v.x), J.qp, &r));
        o.y = static_cast<uint32_t>(quantize_f32(__uint_as_float(v.y), J.qp, &r));
        o.z = static_cast<uint32_t>(quantize_f32(__uint_as_float(v.z), J.qp, &r));
        o.w = static_cast<uint32_t>(quantize_f32(__uint_as_float(v.w), J.qp, &r));
        d4[q] = o;
      }
      return;
    }
    for (uint32_t l = threadIdx.x; l < ne; l += kBlock) {
      uint32_t r = 0;
      const uint32_t c = static_cast<uint32_t>(job_code(J, e0 + l, &r));
      uint8_t* s = stage + mis + 4 * l;
      s[0] = static_cast<uint8_t>(c);
      s[1] = static_cast<uint8_t>(c >> 8);
      s[2] = static_cast<uint8_t>(c >> 16);
      s[3] = static_cast<uint8_t>(c >> 24);
    }
    __syncthreads();
    copy_out_staged(dst, stage, 4ull * ne);
    return;
  }

  if (codec == EMBC_CODEC_VLZ) {  // token stream (vlz.hpp:111-125)
    if (!fits) return;
    uint8_t* dst = pay + pre / 8;
    if constexpr (prestage) {
      TS(4);
      copy_out_shifted(dst, stage, 0, pst);
    } else {
      const uint32_t mis = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(dst) & 15);
      const uint32_t tot = stage_vlz(mis);
      TS(4);
      copy_out_staged(dst, stage, tot);
    }
    return;
  }

  // huffman bitstream, MSB-first (bitstream.hpp:32-51)
  uint8_t* bstream = pay + book_bytes;
  if (first && fits) {  // the serialized codebook (huffman.hpp:202-209)
    const uint8_t* bk = a.books + static_cast<uint64_t>(J.hjob) * a.book_stride;
    for (uint64_t k = threadIdx.x; k < book_bytes; k += kBlock) pay[k] = bk[k];
  }
  uint8_t* dst = bstream + (pre >> 3);
  const uint32_t b0 = static_cast<uint32_t>(pre & 7);
  // phase 2: staged from byte 0 before the job look-back; else aligned with dst
  const uint32_t mis = prestage ? 0u : static_cast<uint32_t>(reinterpret_cast<uintptr_t>(dst) & 15);
  uint32_t nbytes_stage;
  if constexpr (prestage) nbytes_stage = pst;
  else nbytes_stage = stage_huff(mis);
  const uint32_t endbit = 8 * mis + b0 + static_cast<uint32_t>(my_bits);
  TS(4);
  const uint32_t nbytes = nbytes_stage - mis;  // output bytes touched by this tile
  const bool head_shared = b0 != 0;
  const bool tail_shared = !last && (endbit & 7) != 0;
  if (fits) {
    const uint32_t lo = head_shared ? 1 : 0, hi = nbytes - (tail_shared ? 1 : 0);
    if constexpr (prestage) {
      if (hi > lo) copy_out_shifted(dst + lo, stage, lo, hi - lo);
    } else {
      copy_range(dst, stage, mis, lo, hi);
    }
  }
  // bytes shared with the neighbouring tiles: the second of the two to arrive
  // writes the OR of both halves and re-arms the slot (kept zero between calls)
  if (threadIdx.x == 0) {
    if (head_shared) {
      const uint32_t mine = stage[mis];
      const uint32_t old = atomicOr(&a.edge_slot[tid], 0x100u | mine);
      if (old & 0x200u) {
        if (fits) dst[0] = static_cast<uint8_t>((old | mine) & 0xFF);
        a.edge_slot[tid] = 0;
      }
    }
    if (tail_shared) {
      const uint32_t mine = stage[nbytes_stage - 1];
      const uint32_t old = atomicOr(&a.edge_slot[tid + 1], 0x200u | mine);
      if (old & 0x100u) {
        if (fits) dst[nbytes - 1] = static_cast<uint8_t>((old | mine) & 0xFF);
        a.edge_slot[tid + 1] = 0;
      }
    }
  }
}

template <int PHASE>
__global__ void __launch_bounds__(kBlock, 4) k_emit(EmitArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  // tile = block index: the look-back (phase 2) only waits on lower tiles,
  // dispatched first
  emit_tile<PHASE, false>(a, blockIdx.x, smem);
}

// Single-launch encode of small calls: E1 then E2 (phase 2) in the same CTA,
// the tile's codes kept in shared memory.  Waits, all on earlier tickets
// except one: vlz tiles on the window's hashes, E2 on earlier tiles' sizes,
// and huffman tiles on their job's codebook, built by whichever tile of the
// job finishes E1 last -- tickets are dealt in job order, so a job's tiles
// hold consecutive tickets and the host only picks this kernel when every
// job's tiles fit on the GPU at once.
struct FusedArgs {
  StatsArgs s;
  EmitArgs e;
};

__global__ void __launch_bounds__(kBlock, 4) k_encode(FusedArgs f) {
  extern __shared__ __align__(16) uint8_t smem[];
  // tile = block index: every wait is on a lower tile (look-backs, vlz hash
  // windows) or on a codebook whose builder is resident (all tiles fit at once)
  const uint32_t tid = blockIdx.x;
  EMBC_DBG(dbg_kspan_begin());
  stats_tile<true>(f.s, tid, smem);
  const uint32_t jid = f.e.tiles[tid].job;
  if (f.e.jobs[jid].codec == EMBC_CODEC_HUFFMAN) {
    if (threadIdx.x == 0) {
      uint32_t delay = 32;
      while (!*reinterpret_cast<volatile uint32_t*>(&f.e.st[jid].flags)) {
        __nanosleep(delay);
        delay = min(delay * 2, kPollMaxNs);
      }
      __threadfence();
    }
    __syncthreads();
  }
  emit_tile<2, true>(f.e, tid, smem);
  EMBC_DBG(dbg_kspan_end(f.e.ntiles));
}

}  // namespace embc_dev

// ===========================================================================
// host orchestration
// ===========================================================================
namespace embc_host {

using namespace embc_dev;

// An encode call with no jobs: the packed layout's rank count (0) and the total.
__global__ void k_empty_call(uint8_t* out, uint64_t* d_total, uint64_t total) {
  if (threadIdx.x < total) out[threadIdx.x] = 0;
  if (threadIdx.x == 0 && d_total) *d_total = total;
}

static inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Carve {
  size_t off = 0;
  template <typename T>
  size_t take(size_t count, size_t align = 16) {
    off = align_up(off, align);
    const size_t o = off;
    off += sizeof(T) * count;
    return o;
  }
};

static uint32_t pick_tile_rows(uint32_t dim, uint64_t total_values) {
  // ~2 tiles per SM on a 148-SM part, 1K..4K values per tile, <= 1024 rows
  uint64_t target = total_values / 296;
  target = std::max<uint64_t>(1024, std::min<uint64_t>(kTileVals, target));
  uint64_t rows = std::max<uint64_t>(1, target / std::max<uint32_t>(dim, 1));
  rows = std::min<uint64_t>(rows, kMaxTileRows);
  while (rows > 1 && rows * dim > kTileVals) --rows;
  return static_cast<uint32_t>(rows);
}

uint64_t encode_bound(const embc_job* jobs, uint32_t njobs, int layout) {
  uint64_t b = layout == EMBC_LAYOUT_PACKED ? 4 + 16ull * njobs : 0;
  for (uint32_t j = 0; j < njobs; ++j) {
    const uint64_t N = static_cast<uint64_t>(jobs[j].dim) * jobs[j].n;
    uint64_t p;
    if (jobs[j].codec == EMBC_CODEC_RAW) p = 4 * N;
    else if (jobs[j].codec == EMBC_CODEC_VLZ) p = static_cast<uint64_t>(jobs[j].n) * std::max<uint64_t>(4, 1 + 5ull * jobs[j].dim);
    else p = 12 + 5 * std::min<uint64_t>(N, kHistCap) + 4 * N + 1;
    b += (layout == EMBC_LAYOUT_PAYLOAD ? 0 : kHeader) + p;
  }
  return b;
}

static embc_status encode_impl(embc_ctx* ctx, const embc_job* hj, uint32_t njobs, int layout,
                               uint8_t* d_out, uint64_t cap, uint64_t* d_offsets,
                               uint64_t* d_lengths, uint8_t* d_meta, uint64_t* d_total,
                               cudaStream_t stream, unsigned long long* d_stats);

embc_status encode(embc_ctx* ctx, const embc_job* hj, uint32_t njobs, int layout, uint8_t* d_out,
                   uint64_t cap, uint64_t* d_offsets, uint64_t* d_lengths, uint8_t* d_meta,
                   uint64_t* d_total, cudaStream_t stream) {
  return encode_impl(ctx, hj, njobs, layout, d_out, cap, d_offsets, d_lengths, d_meta, d_total,
                     stream, nullptr);
}

// match_stats (vlz.hpp:162-168): the E1/E2 dedup decisions of one job, counted.
embc_status match_stats(embc_ctx* ctx, const int32_t* d_codes, uint32_t dim, uint32_t n,
                        uint32_t window, uint64_t* h_lit, uint64_t* h_ref, cudaStream_t stream) {
  if (window < 1 || window > kMaxWindow)  // VlzConfig::validate (vlz.hpp:39-43)
    return set_error(ctx, EMBC_ERR_VALUE, EMBC_R_BAD_WINDOW, 0, 0, 0, window,
                     format_message(EMBC_R_BAD_WINDOW, 0, 0, window, 0.0));
  if (dim == 0 && n > 0)
    return set_error(ctx, EMBC_ERR_VALUE, EMBC_R_DIM0, 0, 0, 0, 0, "embedding batch dim must be >= 1");
  *h_lit = 0;
  *h_ref = 0;
  if (n == 0) return EMBC_OK;
  embc_job j{};
  j.src = d_codes;
  j.dim = dim;
  j.n = n;
  j.eb = 0.01;
  j.window = window;
  j.codec = EMBC_CODEC_VLZ;
  j.src_kind = EMBC_SRC_I32;
  unsigned long long* d_cnt = nullptr;
  cudaError_t ce = cudaMallocAsync(&d_cnt, 16, stream);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "match_stats");
  cudaMemsetAsync(d_cnt, 0, 16, stream);
  embc_status st = encode_impl(ctx, &j, 1, EMBC_LAYOUT_PAYLOAD, nullptr, 0, nullptr, nullptr,
                               nullptr, nullptr, stream, d_cnt);
  unsigned long long h[2] = {0, 0};
  if (st == EMBC_OK) {
    ce = cudaMemcpyAsync(h, d_cnt, 16, cudaMemcpyDeviceToHost, stream);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(stream);
    if (ce != cudaSuccess) st = cuda_fail(ctx, ce, "match_stats readback");
  }
  cudaFreeAsync(d_cnt, stream);
  *h_lit = h[0];
  *h_ref = h[1];
  return st;
}

static embc_status encode_impl(embc_ctx* ctx, const embc_job* hj, uint32_t njobs, int layout,
                               uint8_t* d_out, uint64_t cap, uint64_t* d_offsets,
                               uint64_t* d_lengths, uint8_t* d_meta, uint64_t* d_total,
                               cudaStream_t stream, unsigned long long* d_stats) {
  // ---- argument validation (host-known, raised before any device work in the
  //      reference as well: ErrorBound ctor at container.hpp:308, check_shape)
  ctx->job_eb.assign(njobs, 0.0);
  ctx->job_window.assign(njobs, 0);
  if (njobs == 0) {
    // pack([]) is the 4-byte rank count 0 (container.hpp:242-256); the other
    // layouts are empty.  Written on the stream like any other output.
    const uint64_t total = layout == EMBC_LAYOUT_PACKED ? 4 : 0;
    if (total && (cap < total || !d_out))
      return set_error(ctx, EMBC_ERR_CAPACITY, EMBC_R_CAPACITY, 0, 0, total, cap,
                       format_message(EMBC_R_CAPACITY, 0, total, cap, 0.0));
    if (total || d_total) {
      k_empty_call<<<1, 32, 0, stream>>>(total ? d_out : nullptr, d_total, total);
      cudaError_t ce = cudaGetLastError();
      if (ce != cudaSuccess) return cuda_fail(ctx, ce, "empty encode");
    }
    return EMBC_OK;
  }
  std::vector<DJob> jobs(njobs);
  std::vector<DTile> tiles;
  uint64_t total_values = 0, total_rows = 0;
  for (uint32_t j = 0; j < njobs; ++j) total_values += static_cast<uint64_t>(hj[j].dim) * hj[j].n;
  uint32_t nhuff = 0;
  uint64_t hist_entries = 0;
  bool host_abort = false;
  for (uint32_t j = 0; j < njobs; ++j) {
    const embc_job& in = hj[j];
    ctx->job_eb[j] = in.eb;
    ctx->job_window[j] = in.window;
    if (!(std::isfinite(in.eb) && in.eb > 0.0))
      return set_error(ctx, EMBC_ERR_VALUE, EMBC_R_BAD_EB, j, 0, 0, 0,
                       "error bound must be finite and > 0, got " + fmt_double(in.eb));
    if (in.codec > EMBC_CODEC_HUFFMAN || in.src_kind > EMBC_SRC_I32 || (!in.src && in.n && in.dim))
      return set_error(ctx, EMBC_ERR_ARGUMENT, 0, j, 0, 0, 0, "invalid job descriptor");
    if (in.dim == 0)
      return set_error(ctx, EMBC_ERR_VALUE, EMBC_R_DIM0, j, 0, 0, 0, "embedding batch dim must be >= 1");
    if (in.dim > kMaxRowVals)
      return set_error(ctx, EMBC_ERR_UNSUPPORTED, 0, j, 0, 0, 0, "dim > 8192 is outside the GPU tile envelope");
    DJob& J = jobs[j];
    J.src = in.src;
    J.dim = in.dim;
    J.n = in.n;
    J.N = static_cast<uint64_t>(in.dim) * in.n;
    if (J.N >= (1ull << 32))
      return set_error(ctx, EMBC_ERR_UNSUPPORTED, 0, j, 0, 0, 0, "chunk of >= 2^32 values");
    J.window = in.window;
    J.window_ok = in.window >= 1 && in.window <= kMaxWindow;
    J.codec = in.codec;
    J.src_kind = in.src_kind;
    J.header = layout == EMBC_LAYOUT_PAYLOAD ? 0 : kHeader;
    J.qp.eb = in.eb;
    J.qp.w = 2.0 * in.eb;
    const double rw = 1.0 / J.qp.w;
    J.qp.rw = static_cast<float>(rw);
    J.qp.fast = (rw >= 0x1.0p-100 && rw <= 0x1.0p100) ? 1 : 0;
    J.fd = make_fastdiv(in.dim);
    J.row_base = total_rows;
    total_rows += in.n;
    J.hjob = -1;
    J.hist_cap = 0;
    if (in.codec == EMBC_CODEC_HUFFMAN) {
      J.hjob = static_cast<int32_t>(nhuff++);
      J.hist_cap = std::min<uint64_t>(std::max<uint64_t>(J.N, 1), kHistCap);  // bound on distinct symbols
      hist_entries += kWin;
    }
    if (in.codec == EMBC_CODEC_VLZ && !J.window_ok) host_abort = true;
    J.tile_rows = pick_tile_rows(in.dim, total_values);
    J.tile0 = static_cast<uint32_t>(tiles.size());
    for (uint32_t r = 0; r < in.n; r += J.tile_rows) {
      DTile t{};
      t.job = j;
      t.row0 = r;
      t.rows = std::min<uint32_t>(J.tile_rows, in.n - r);
      tiles.push_back(t);
    }
    if (in.n == 0) tiles.push_back(DTile{j, 0, 0, 0});  // every job publishes through one tile
    J.ntiles = static_cast<uint32_t>(tiles.size()) - J.tile0;
  }
  const uint32_t ntiles = static_cast<uint32_t>(tiles.size());
  uint32_t vals_max = 1, rows_max = 1;
  for (const DTile& t : tiles) {
    vals_max = std::max(vals_max, t.rows * jobs[t.job].dim);
    rows_max = std::max(rows_max, t.rows);
  }
  uint64_t book_cap = 1;
  for (uint32_t j = 0; j < njobs; ++j)
    if (jobs[j].codec == EMBC_CODEC_HUFFMAN) book_cap = std::max<uint64_t>(book_cap, jobs[j].hist_cap);
  uint64_t p2cap = 1;
  while (p2cap < book_cap) p2cap <<= 1;
  const uint64_t book_stride = align_up(12 + 5 * book_cap, 16);
  const bool big_books = p2cap > kSmemBook;

  // ---- scratch carve
  Carve cv;
  const size_t o_jobs = cv.take<DJob>(njobs);
  const size_t o_tiles = cv.take<DTile>(ntiles);
  const size_t o_st = cv.take<JobState>(njobs);
  const size_t o_flags = cv.take<uint32_t>(8);
  const size_t o_hready = cv.take<uint32_t>(ntiles + 1);
  const size_t o_tstat = cv.take<unsigned long long>(ntiles + 1);
  const size_t o_jstat = cv.take<unsigned long long>(kJobStride * (njobs + 1), 128);
  const size_t o_slot = cv.take<uint32_t>(ntiles + 1);
  const size_t o_zero = o_hready;    // [hready .. edge slots] start at zero every call
  const size_t host_bytes = cv.off;  // everything above is uploaded from the host
  const size_t o_info = cv.take<uint64_t>(total_rows + 1);
  const size_t o_rdec = cv.take<uint32_t>(total_rows + 1);
  const size_t o_tbits = cv.take<uint64_t>(ntiles + 1);
  const size_t o_toff = cv.take<uint64_t>(ntiles + 1);
  const size_t o_jstart = cv.take<uint64_t>(njobs + 1);
  hist_entries += kWidePool;  // [nhuff windows | wide pool], LUT mirrors the layout
  const size_t o_lut = cv.take<uint64_t>(hist_entries + 1);
  const size_t o_books = cv.take<uint8_t>(book_stride * std::max<uint32_t>(nhuff, 1));
  static const uint32_t fused_max = getenv("EMBC_FUSED_MAX") ? atoi(getenv("EMBC_FUSED_MAX")) : 1024;
  const bool two_pass = !d_stats && ntiles > fused_max;
  const bool keep_hist = two_pass && nhuff > 0;  // E1 keeps huffman tile histograms for E2's sizes pass
  const size_t o_thist = keep_hist ? cv.take<uint32_t>(static_cast<uint64_t>(ntiles) * kTileHist) : 0;
  const size_t o_thr = keep_hist ? cv.take<int2>(ntiles) : 0;
  size_t o_gkey = 0, o_gwgt = 0, o_gpar = 0;
  if (big_books) {
    o_gkey = cv.take<uint64_t>(p2cap * nhuff);
    o_gwgt = cv.take<uint64_t>(2 * p2cap * nhuff);
    o_gpar = cv.take<int32_t>(2 * p2cap * nhuff);
  }
  cudaError_t ce = ensure_scratch(ctx, cv.off);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "scratch allocation");
  uint8_t* hs = nullptr;
  int slot = -1;
  ce = stage_acquire(ctx, host_bytes, stream, &hs, &slot);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "staging allocation");
  ce = ensure_hist(ctx, hist_entries);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "histogram allocation");

  // ---- upload descriptors + initial job state in one copy
  std::memcpy(hs + o_jobs, jobs.data(), sizeof(DJob) * njobs);
  std::memcpy(hs + o_tiles, tiles.data(), sizeof(DTile) * ntiles);
  for (uint32_t j = 0; j < njobs; ++j) {
    JobState s{};
    s.cmin = INT_MAX;
    s.cmax = INT_MIN;
    s.err = ~0ull;
    // an invalid vlz window is the reference's ValueError from vlz_encode,
    // raised after quantization (container.hpp:121, :135) -> stage-2 key
    if (jobs[j].codec == EMBC_CODEC_VLZ && !jobs[j].window_ok)
      s.err = err_key(0, EMBC_R_BAD_WINDOW) | (1ull << 63);
    std::memcpy(hs + o_st + sizeof(JobState) * j, &s, sizeof(JobState));
  }
  uint32_t flags0[8] = {host_abort ? JF_ABORT : 0u, 0, 0, 0, 0, 0, 0, 0};
  std::memcpy(hs + o_flags, flags0, sizeof(flags0));
  std::memset(hs + o_zero, 0, host_bytes - o_zero);
  uint8_t* d = ctx->d_scratch;
  ce = stage_upload(ctx, d, hs, host_bytes, slot, stream);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "descriptor upload");

  StatsArgs sa{};
  sa.jobs = reinterpret_cast<const DJob*>(d + o_jobs);
  sa.tiles = reinterpret_cast<const DTile*>(d + o_tiles);
  sa.st = reinterpret_cast<JobState*>(d + o_st);
  sa.row_info = reinterpret_cast<uint64_t*>(d + o_info);
  sa.tile_status = reinterpret_cast<unsigned long long*>(d + o_tstat);
  sa.job_status = reinterpret_cast<unsigned long long*>(d + o_jstat);
  sa.edge_slot = reinterpret_cast<uint32_t*>(d + o_slot);
  sa.book.hist = reinterpret_cast<uint32_t*>(ctx->d_hist);
  sa.book.lut = reinterpret_cast<uint64_t*>(d + o_lut);
  sa.book.books = d + o_books;
  sa.book.book_stride = book_stride;
  if (big_books) {
    sa.book.gs.key = reinterpret_cast<uint64_t*>(d + o_gkey);
    sa.book.gs.wgt = reinterpret_cast<uint64_t*>(d + o_gwgt);
    sa.book.gs.parent = reinterpret_cast<int32_t*>(d + o_gpar);
  }
  sa.book.gs_stride = p2cap;
  sa.book.nhuff = nhuff;
  sa.book.flags = reinterpret_cast<uint32_t*>(d + o_flags);
  // small calls: one fused E2 pass (sizes, decoupled look-back, bytes) -- the
  // look-back is cheap when every tile is resident at once -- with the vlz
  // matching in E1; large calls: E2 sizes (matching included) + layout, then
  // bytes, with no waiting at all
  const bool fused = !d_stats && ntiles <= fused_max;
  sa.match = fused || d_stats ? 1u : 0u;
  sa.hist_off = stats_codes_bytes(vals_max, rows_max);
  sa.tile_hist = keep_hist ? reinterpret_cast<uint32_t*>(d + o_thist) : nullptr;
  sa.tile_hr = keep_hist ? reinterpret_cast<int2*>(d + o_thr) : nullptr;
  sa.row_dec = reinterpret_cast<uint32_t*>(d + o_rdec);
  sa.hready = reinterpret_cast<uint32_t*>(d + o_hready);
  sa.d_stats = d_stats;
  uint32_t stats_aux = nhuff ? kWin * 4 : 0;
  {
    uint32_t wmax = 0;
    bool any_vlz = false;
    for (uint32_t j = 0; j < njobs; ++j)
      if (jobs[j].codec == EMBC_CODEC_VLZ && jobs[j].window_ok) {
        any_vlz = true;
        wmax = std::max(wmax, jobs[j].window);
      }
    if (any_vlz && sa.match) {
      sa.rows_cap = rows_max;
      sa.hash_cap = static_cast<uint32_t>(std::min<uint64_t>(kHashStage, static_cast<uint64_t>(wmax) + rows_max));
      sa.chain_bytes = 4 * 2048 + 2 * sa.hash_cap;
      stats_aux = std::max<uint32_t>(stats_aux, 4 * sa.hash_cap + 16 * sa.rows_cap + sa.chain_bytes);
    }
  }
  const uint32_t stats_smem = sa.hist_off + stats_aux;

  EmitArgs ea{};
  ea.jobs = sa.jobs;
  ea.tiles = sa.tiles;
  ea.st = sa.st;
  ea.row_info = sa.row_info;
  ea.tile_status = sa.tile_status;
  ea.job_status = sa.job_status;
  ea.edge_slot = sa.edge_slot;
  ea.lut = sa.book.lut;
  ea.books = sa.book.books;
  ea.book_stride = book_stride;
  ea.flags = sa.book.flags;
  ea.njobs = njobs;
  ea.ntiles = ntiles;
  ea.layout = layout;
  ea.out = d_out;
  ea.cap = cap;
  ea.d_offsets = d_offsets;
  ea.d_lengths = d_lengths;
  ea.d_meta = d_meta;
  ea.d_total = d_total;
  ea.err = ctx->d_err;
  ea.d_stats = d_stats;
  bool has_vlz = false, has_huf = false;
  for (uint32_t j = 0; j < njobs; ++j) {
    has_vlz |= jobs[j].codec == EMBC_CODEC_VLZ;
    has_huf |= jobs[j].codec == EMBC_CODEC_HUFFMAN;
  }
  ea.stage_off = emit_codes_bytes(vals_max, rows_max);
  ea.aux_off = ea.stage_off + emit_stage_bytes(vals_max, rows_max, has_vlz);
  ea.rows_cap = rows_max;
  // aux: [huffman LUT stage | vlz: hash stage (phase 0) ][vlz: match offset,
  // token bytes, (phase 0:) candidate, pending list, miss per row]
  uint32_t wmax = 0;
  for (uint32_t j = 0; j < njobs; ++j)
    if (jobs[j].codec == EMBC_CODEC_VLZ) wmax = std::max(wmax, jobs[j].window);
  const uint32_t per_row = fused ? 8 : 20;
  ea.hash_cap = has_vlz && !fused ? static_cast<uint32_t>(std::min<uint64_t>(kHashStage, static_cast<uint64_t>(wmax) + rows_max)) : 0;
  uint32_t aux_bytes = ea.hash_cap * 4 + ea.rows_cap * per_row;
  if (has_huf) aux_bytes = std::max<uint32_t>(aux_bytes, 8 * kLutStage + ea.rows_cap * 8);
  ea.hash_cap = (aux_bytes - ea.rows_cap * per_row) / 4;  // any slack widens the hash stage
  const uint32_t emit_smem = ea.aux_off + aux_bytes;
  ea.row_dec = reinterpret_cast<uint32_t*>(d + o_rdec);
  ea.tile_bits = reinterpret_cast<uint64_t*>(d + o_tbits);
  ea.tile_off = reinterpret_cast<uint64_t*>(d + o_toff);
  ea.job_start = reinterpret_cast<uint64_t*>(d + o_jstart);
  ea.done = sa.book.flags + CF_TICKET;  // zeroed by the upload
  ea.tile_hist = sa.tile_hist;
  ea.tile_hr = sa.tile_hr;
  ea.phase = 2;
  // small calls whose tiles all fit on the GPU at once: E1 + E2 in one launch
  // (k_encode), the codes kept in shared memory.  Layout: codes | E1 scratch
  // (histogram window, vlz matching, codebook build) overlapping E2's stage + aux
  if (fused) {
    uint32_t e1 = nhuff ? std::max<uint32_t>(kWin * 4, kSmemBook * 32) : 0;
    if (sa.match && sa.hash_cap) e1 = std::max<uint32_t>(e1, 4 * sa.hash_cap + 16 * sa.rows_cap + sa.chain_bytes);
    const uint32_t merged_smem = ea.stage_off + std::max<uint32_t>(e1, emit_smem - ea.stage_off);
    bool merged = merged_smem <= kEncodeSmemMax;
    if (merged) {
      int per_sm = 0, nsm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_encode, kBlock, merged_smem) != cudaSuccess ||
          cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device) != cudaSuccess) {
        cudaGetLastError();
        per_sm = 0;
      }
      // every tile co-resident on an idle GPU; and since the only wait on a
      // later ticket is within one job (its codebook), a job that fits in one
      // CTA per SM still progresses when other work holds most of the GPU
      uint32_t max_job_tiles = 0;
      for (uint32_t j = 0; j < njobs; ++j) max_job_tiles = std::max(max_job_tiles, jobs[j].ntiles);
      merged = static_cast<uint64_t>(ntiles) <= static_cast<uint64_t>(per_sm) * nsm &&
               max_job_tiles <= static_cast<uint32_t>(nsm);
    }
    static const bool no_merge = getenv("EMBC_NO_MERGE") != nullptr;
    if (merged && !no_merge) {
      FusedArgs f;
      sa.hist_off = ea.stage_off;
      f.s = sa;
      f.e = ea;
      EMBC_TIMED(ctx, "k_encode", stream, k_encode<<<ntiles, kBlock, merged_smem, stream>>>(f));
      ce = cudaGetLastError();
      if (ce != cudaSuccess) return cuda_fail(ctx, ce, "encode launch");
      return EMBC_OK;
    }
  }
  EMBC_TIMED(ctx, "k_stats", stream, k_stats<<<ntiles, kBlock, stats_smem, stream>>>(sa));
  // small calls: one fused pass (sizes, decoupled look-back, bytes) -- the
  // look-back is cheap when every tile is resident at once; large calls: sizes
  // + layout, then bytes, with no waiting at all
  if (d_stats) {
    // match_stats: the counts come from E1
  } else if (fused) {
    ea.phase = 2;
    EMBC_TIMED(ctx, "k_emit", stream, k_emit<2><<<ntiles, kBlock, emit_smem, stream>>>(ea));
  } else {
    ea.phase = 0;
    EMBC_TIMED(ctx, "k_sizes", stream, k_emit<0><<<ntiles, kBlock, emit_smem, stream>>>(ea));
    ea.phase = 1;
    EMBC_TIMED(ctx, "k_emit", stream, k_emit<1><<<ntiles, kBlock, emit_smem, stream>>>(ea));
  }
  ce = cudaGetLastError();
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "encode launch");
  return EMBC_OK;
}

cudaError_t encode_set_attributes() {
  cudaError_t e = cudaFuncSetAttribute(k_emit<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kEmitSmemMax);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_emit<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kEmitSmemMax);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_emit<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kEmitSmemMax);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_encode, cudaFuncAttributeMaxDynamicSharedMemorySize, kEncodeSmemMax);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_stats, cudaFuncAttributeMaxDynamicSharedMemorySize, kStatsSmemMax);
}

}  // namespace embc_host
