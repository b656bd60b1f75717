// encode.cu -- sm_100a compression pipeline: quantize -> (vlz dedup | huffman
// | raw) -> chunk container -> packed send buffer, for a batch of jobs in one
// launch sequence with no host synchronisation (graph-capturable).
//
// Mirrors embc::encode_chunks + embc::pack (container.hpp:119-142, :242-256,
// :304-311).  Kernels:
//   K1 k_quant_stats  quantize every tile, first-failure record, per-row
//                      hash + literal token length (vlz), code range (huffman)
//   K1b k_huff_hist    dense code histogram over [cmin, cmax]   (huffman.hpp:122-128)
//   K2 k_huff_book     two-queue Huffman lengths + canonical codes (huffman.hpp:49-120, :165-186)
//   K3 k_sizes         vlz match decisions (vlz.hpp:86-103) + per-tile output sizes
//   K4 k_layout        chunk offsets (scan, job order), headers, pack table, metadata
//   K5 k_emit          raw / vlz token / huffman bitstream bytes
//   K6 k_huff_edges    OR together the bitstream bytes shared by adjacent tiles
#include <cuda_runtime.h>
#include <limits.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "embc_internal.h"

namespace embc_dev {

// ---------------------------------------------------------------------------
// element access
// ---------------------------------------------------------------------------
__device__ __forceinline__ int32_t job_code(const DJob& J, uint64_t e, uint32_t* reason) {
  if (J.src_kind == EMBC_SRC_F32) {
    const float x = __ldg(static_cast<const float*>(J.src) + e);
    return quantize_f32(x, J.qp, reason);
  }
  return __ldg(static_cast<const int32_t*>(J.src) + e);
}

__device__ __forceinline__ void atomic_min_u64(unsigned long long* p, unsigned long long v) {
  if (v != ~0ull) atomicMin(p, v);
}

// Block min-reduction of a failure key into the job state.
__device__ __forceinline__ void publish_err(unsigned long long* dst, unsigned long long v,
                                            unsigned long long* s_tmp) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long n = __shfl_xor_sync(0xffffffffu, v, o);
    v = n < v ? n : v;
  }
  if ((threadIdx.x & 31) == 0 && v != ~0ull) atomicMin(s_tmp, v);
}

// ---------------------------------------------------------------------------
// K1: quantize + per-row statistics
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock) k_quant_stats(const DJob* __restrict__ jobs,
                                                        const DTile* __restrict__ tiles,
                                                        JobState* __restrict__ st,
                                                        uint64_t* __restrict__ row_hash,
                                                        uint32_t* __restrict__ row_lit,
                                                        uint32_t* __restrict__ whist,
                                                        uint32_t hist_smem_off) {
  extern __shared__ __align__(16) uint8_t smem[];
  // huffman jobs: speculative histogram over the window [-kWin/2, kWin/2)
  // (Codebook::build, huffman.hpp:122-128); K2 redoes it for wider alphabets
  uint32_t* shist = reinterpret_cast<uint32_t*>(smem + hist_smem_off);
  __shared__ unsigned long long s_err;
  __shared__ int s_min, s_max;
  const DTile T = tiles[blockIdx.x];
  const DJob& J = jobs[T.job];
  const uint32_t dim = J.dim;
  const uint32_t stride = dim | 1u;
  const bool vlz = J.codec == EMBC_CODEC_VLZ;
  const bool huf = J.codec == EMBC_CODEC_HUFFMAN;
  int32_t* codes = reinterpret_cast<int32_t*>(smem);
  if (threadIdx.x == 0) {
    s_err = ~0ull;
    s_min = INT_MAX;
    s_max = INT_MIN;
  }
  if (huf)
    for (uint32_t b = threadIdx.x; b < kWin; b += blockDim.x) shist[b] = 0;
  __syncthreads();
  bool lwide = false;

  const uint64_t e0 = static_cast<uint64_t>(T.row0) * dim;
  const uint32_t ne = T.rows * dim;
  unsigned long long lerr = ~0ull;
  int lmin = INT_MAX, lmax = INT_MIN;
  if (J.src_kind == EMBC_SRC_F32) {
    const float* x = static_cast<const float*>(J.src) + e0;
    const QParams qp = J.qp;
    for (uint32_t l = threadIdx.x; l < ne; l += blockDim.x) {
      uint32_t reason = 0;
      const int32_t c = quantize_f32(__ldg(x + l), qp, &reason);
      if (reason) lerr = min(lerr, static_cast<unsigned long long>(err_key(e0 + l, reason)));
      lmin = min(lmin, c);
      lmax = max(lmax, c);
      if (huf) {
        const uint32_t b = static_cast<uint32_t>(c + static_cast<int32_t>(kWin / 2));
        if (b < kWin) atomicAdd(&shist[b], 1u);
        else lwide = true;
      }
      if (vlz) {
        const uint32_t r = fdiv(l, J.fd);
        codes[r * stride + (l - r * dim)] = c;
      }
    }
  } else {
    const int32_t* x = static_cast<const int32_t*>(J.src) + e0;
    for (uint32_t l = threadIdx.x; l < ne; l += blockDim.x) {
      const int32_t c = __ldg(x + l);
      lmin = min(lmin, c);
      lmax = max(lmax, c);
      if (huf) {
        const uint32_t b = static_cast<uint32_t>(c + static_cast<int32_t>(kWin / 2));
        if (b < kWin) atomicAdd(&shist[b], 1u);
        else lwide = true;
      }
      if (vlz) {
        const uint32_t r = fdiv(l, J.fd);
        codes[r * stride + (l - r * dim)] = c;
      }
    }
  }
  publish_err(&st[T.job].err, lerr, &s_err);
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
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_err != ~0ull) atomicMin(&st[T.job].err, s_err);
    if (huf) {
      atomicMin(&st[T.job].cmin, s_min);
      atomicMax(&st[T.job].cmax, s_max);
    }
  }
  if (huf) {
    const bool wide = __syncthreads_or(lwide);
    if (wide) {
      if (threadIdx.x == 0) st[T.job].wide = 1;
    } else {
      uint32_t* gh = whist + static_cast<uint64_t>(J.hjob) * kWin;
      for (uint32_t b = threadIdx.x; b < kWin; b += blockDim.x) {
        const uint32_t v = shist[b];
        if (v) atomicAdd(&gh[b], v);
      }
    }
  }
  if (vlz) {
    // Row hash (any function works: equality is verified exactly in K3) and
    // literal token length 1 + sum varint_len(zigzag(c)) (vlz.hpp:115-118).
    for (uint32_t r = threadIdx.x; r < T.rows; r += blockDim.x) {
      const int32_t* row = codes + r * stride;
      uint64_t h = 0xCBF29CE484222325ull;
      uint32_t lit = 1;
      for (uint32_t j = 0; j < dim; ++j) {
        const int32_t c = row[j];
        lit += varint_len(zigzag(c));
        h = (h ^ static_cast<uint32_t>(c)) * 0x100000001B3ull;
      }
      h ^= h >> 29;
      const uint64_t g = J.row_base + T.row0 + r;
      row_hash[g] = h;
      row_lit[g] = lit;
    }
  }
}

// ---------------------------------------------------------------------------
// K2: canonical Huffman codebook per job (one CTA).
// ---------------------------------------------------------------------------
// In-place ascending bitonic sort of n keys (n padded to a power of two with
// ~0 sentinels by the caller); generic pointer: shared or global memory.
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

constexpr uint32_t kBookThreads = 1024;
constexpr uint32_t kSmemBook = 2048;  // symbols handled fully in shared memory

__global__ void __launch_bounds__(kBookThreads) k_huff_book(
    const DJob* __restrict__ jobs, const uint32_t* __restrict__ hjob_list, JobState* __restrict__ st,
    uint32_t* __restrict__ hist, uint64_t* __restrict__ lut, uint8_t* __restrict__ books,
    uint64_t book_stride, BookScratch gs, uint64_t gs_stride, uint32_t nhuff,
    unsigned long long* __restrict__ wide_ctr) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t s_tmp32[33];
  __shared__ unsigned long long s_tmp64[33];
  __shared__ uint32_t s_nsym;
  __shared__ unsigned long long s_cap;
  __shared__ unsigned long long s_woff;
  const uint32_t jid = hjob_list[blockIdx.x];
  const DJob& J = jobs[jid];
  JobState& S = st[jid];
  const uint32_t hj = static_cast<uint32_t>(J.hjob);
  uint32_t* narrow = hist + static_cast<uint64_t>(hj) * kWin;
  if (S.err != ~0ull || J.N == 0) {
    // quantization failed (or nothing to code): leave the window histogram clean
    for (uint32_t b = threadIdx.x; b < kWin; b += blockDim.x) narrow[b] = 0;
    if (J.N == 0 && S.err == ~0ull && threadIdx.x == 0)  // huffman.hpp:229
      S.err = err_key(0, EMBC_R_HUF_EMPTY) | (1ull << 63);
    return;
  }
  const int32_t cmin = S.cmin;
  const uint64_t span = static_cast<uint64_t>(static_cast<int64_t>(S.cmax) - cmin + 1);
  uint32_t* gh;
  if (S.wide) {
    // alphabet wider than the K1 window: histogram over [cmin, cmax] in the
    // wide pool (huffman.hpp:122-128), EMBC_R_RANGE beyond kHistCap
    for (uint32_t b = threadIdx.x; b < kWin; b += blockDim.x) narrow[b] = 0;
    if (threadIdx.x == 0) {
      s_woff = ~0ull;
      if (span <= kHistCap) {
        const unsigned long long o = atomicAdd(wide_ctr, static_cast<unsigned long long>(span));
        if (o + span <= kWidePool) s_woff = o;
      }
    }
    __syncthreads();
    if (s_woff == ~0ull) {
      if (threadIdx.x == 0) {
        S.aux = span;
        S.err = err_key(0, EMBC_R_RANGE) | (1ull << 63);
      }
      return;
    }
    gh = hist + static_cast<uint64_t>(nhuff) * kWin + s_woff;
    for (uint64_t e = threadIdx.x; e < J.N; e += blockDim.x) {
      uint32_t r = 0;
      atomicAdd(&gh[job_code(J, e, &r) - cmin], 1u);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) S.lut_off = static_cast<uint64_t>(nhuff) * kWin + s_woff;
  } else {
    gh = narrow + (cmin + static_cast<int32_t>(kWin / 2));
    if (threadIdx.x == 0) S.lut_off = static_cast<uint64_t>(hj) * kWin + (cmin + static_cast<int32_t>(kWin / 2));
  }
  __syncthreads();

  // 1. compact nonzero bins -> symbols in ascending order (sorted histogram, huffman.hpp:51)
  if (threadIdx.x == 0) s_nsym = 0;
  __syncthreads();
  // first pass: count
  uint32_t cnt = 0;
  for (uint64_t b = threadIdx.x; b < span; b += blockDim.x) cnt += __ldcg(gh + b) != 0;
  const uint32_t nsym = block_sum<uint32_t>(cnt, s_tmp32);

  uint32_t p2 = 1;
  while (p2 < nsym) p2 <<= 1;
  const bool in_smem = p2 <= kSmemBook;
  uint64_t* key = in_smem ? reinterpret_cast<uint64_t*>(smem) : gs.key + hj * gs_stride;
  uint64_t* wgt = in_smem ? key + kSmemBook : gs.wgt + hj * 2 * gs_stride;
  int32_t* parent = in_smem ? reinterpret_cast<int32_t*>(wgt + 2 * kSmemBook)
                            : gs.parent + hj * 2 * gs_stride;

  // second pass: scatter (count << 32 | sym - cmin) keys in symbol order
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
  }
  for (uint32_t i = nsym + threadIdx.x; i < p2; i += blockDim.x) key[i] = ~0ull;
  __syncthreads();

  uint8_t* book = books + hj * book_stride;
  uint64_t* L = lut + S.lut_off;
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
    uint64_t wl = wgt[0];  // weight at the leaf head
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

  // 4. code lengths = leaf depth; first leaf (sorted order) past 32 bits fails
  //    with its depth (huffman.hpp:110-118)
  for (uint32_t i = threadIdx.x; i < nsym; i += blockDim.x) {
    uint32_t depth = 0;
    if (nsym == 1) {
      depth = 1;
    } else {
      for (int32_t p = parent[i]; p != -1; p = parent[p]) ++depth;
    }
    if (depth > 32) atomicMin(&s_cap, (static_cast<unsigned long long>(i) << 32) | depth);
    // canonical sort key: (length, symbol) (huffman.hpp:166-168)
    const uint64_t sym = key[i] & 0xFFFFFFFFull;
    wgt[i] = (static_cast<uint64_t>(depth > 32 ? 63 : depth) << 32) | sym;
  }
  __syncthreads();
  if (s_cap != ~0ull) {
    if (threadIdx.x == 0) {
      S.aux = s_cap & 0xFFFFFFFFull;
      atomicMin(&S.err, err_key(s_cap >> 32, EMBC_R_HUF_LEN_CAP) | (1ull << 63));
    }
    // leave the histogram clean for the next call
    for (uint64_t b = threadIdx.x; b < span; b += blockDim.x) gh[b] = 0;
    return;
  }
  // 5. canonical order (length asc, symbol asc)
  uint64_t* ckey = wgt;  // reuse
  for (uint32_t i = nsym + threadIdx.x; i < p2; i += blockDim.x) ckey[i] = ~0ull;
  __syncthreads();
  if (nsym > 1) bitonic_sort(ckey, p2);

  // 6. canonical code values: code_i = sum_{j<i} 2^(len_i - len_j)  (the closed
  //    form of finalize's shift-and-increment, huffman.hpp:170-181)
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
        bits_local += static_cast<uint64_t>(gh[symoff]) * len;
      }
      carry += tot;
    }
  }
  const unsigned long long bits = block_sum<unsigned long long>(bits_local, s_tmp64);
  // clean histogram for the next call
  for (uint64_t b = threadIdx.x; b < span; b += blockDim.x) gh[b] = 0;
  if (threadIdx.x == 0) {
    st_be(book, J.N, 8);   // u64be symbol_count (huffman.hpp:203)
    st_be(book + 8, nsym, 4);  // u32be entry_count (huffman.hpp:204)
    S.nsym = nsym;
    S.bits = bits;
    S.payload = 12 + 5ull * nsym + (bits + 7) / 8;
  }
}

// ---------------------------------------------------------------------------
// K3: vlz match decisions + per-tile output sizes
// ---------------------------------------------------------------------------
constexpr uint32_t kHashStage = 4096;

__device__ __forceinline__ uint64_t lut_entry(const uint64_t* L, int32_t c, int32_t cmin) {
  return __ldg(L + (c - cmin));
}

// Exact row comparison (the reference's CodeRowEq, vlz.hpp:75-79): one warp
// compares rows a and b of job J.
__device__ __forceinline__ bool warp_rows_equal(const DJob& J, uint32_t a, uint32_t b) {
  const uint32_t lane = threadIdx.x & 31;
  bool eq = true;
  for (uint32_t j = lane; j < J.dim; j += 32) {
    uint32_t r = 0;
    const int32_t ca = job_code(J, static_cast<uint64_t>(a) * J.dim + j, &r);
    const int32_t cb = job_code(J, static_cast<uint64_t>(b) * J.dim + j, &r);
    eq = eq && (ca == cb);
  }
  return __all_sync(0xffffffffu, eq);
}

__device__ __forceinline__ void sizes_tile(const DJob* __restrict__ jobs, const DTile* __restrict__ tiles,
                                           const uint32_t* __restrict__ tile_list,
                                           const JobState* __restrict__ st,
                                           const uint64_t* __restrict__ row_hash,
                                           const uint32_t* __restrict__ row_lit, uint32_t* __restrict__ row_off,
                                           const uint64_t* __restrict__ lut, uint64_t* __restrict__ tile_sum,
                                           uint8_t* smem) {
  __shared__ unsigned long long s_tmp64[33];
  const uint32_t tid = tile_list[blockIdx.x];
  const DTile T = tiles[tid];
  const DJob& J = jobs[T.job];
  const JobState& S = st[T.job];
  if (S.err != ~0ull) return;
  uint64_t local = 0;
  if (J.codec == EMBC_CODEC_VLZ) {
    const uint32_t W = J.window;
    const uint32_t lo = T.row0 > W ? T.row0 - W : 0;
    const uint32_t nh = T.row0 + T.rows - lo;
    const bool staged = nh <= kHashStage;
    uint64_t* sh = reinterpret_cast<uint64_t*>(smem);
    const uint64_t* gh = row_hash + J.row_base;
    if (staged) {
      for (uint32_t k = threadIdx.x; k < nh; k += blockDim.x) sh[k] = gh[lo + k];
    }
    __syncthreads();
    for (uint32_t rb = 0; rb < T.rows; rb += blockDim.x) {
      const uint32_t r = rb + threadIdx.x;
      const bool active = r < T.rows;
      const uint32_t i = T.row0 + r;
      const uint64_t h = active ? (staged ? sh[i - lo] : gh[i]) : 0;
      const uint32_t kmax = active ? min(W, i) : 0;
      uint32_t k = 1;
      uint32_t found = 0;  // offset of the verified match, 0 = literal
      bool searching = active;
      // advance to the next hash candidate
      // nearest candidate first; four independent hash loads per step
      auto next = [&]() {
        while (k + 3 <= kmax) {
          const uint32_t j = i - k;
          uint64_t h0, h1, h2, h3;
          if (staged) {
            h0 = sh[j - lo];
            h1 = sh[j - 1 - lo];
            h2 = sh[j - 2 - lo];
            h3 = sh[j - 3 - lo];
          } else {
            h0 = gh[j];
            h1 = gh[j - 1];
            h2 = gh[j - 2];
            h3 = gh[j - 3];
          }
          if (h0 == h) return true;
          if (h1 == h) { k += 1; return true; }
          if (h2 == h) { k += 2; return true; }
          if (h3 == h) { k += 3; return true; }
          k += 4;
        }
        while (k <= kmax) {
          const uint32_t j = i - k;
          const uint64_t hj = staged ? sh[j - lo] : gh[j];
          if (hj == h) return true;
          ++k;
        }
        return false;
      };
      bool have = searching && next();
      if (!have) searching = false;
      // warp-cooperative exact verification of pending candidates
      for (;;) {
        const uint32_t pend = __ballot_sync(0xffffffffu, searching && have);
        if (!pend) break;
        uint32_t m = pend;
        bool resolved_me = false, eq_me = false;
        while (m) {
          const int src = __ffs(m) - 1;
          m &= m - 1;
          const uint32_t ii = __shfl_sync(0xffffffffu, i, src);
          const uint32_t jj = __shfl_sync(0xffffffffu, i - k, src);
          const bool eq = warp_rows_equal(J, ii, jj);
          if ((threadIdx.x & 31) == static_cast<uint32_t>(src)) {
            resolved_me = true;
            eq_me = eq;
          }
        }
        if (resolved_me) {
          if (eq_me) {
            found = k;
            searching = false;
          } else {
            ++k;  // hash collision: keep looking further back
            have = next();
            if (!have) searching = false;
          }
        }
      }
      if (active) {
        row_off[J.row_base + i] = found;
        local += found ? 1u + varint_len(found) : row_lit[J.row_base + i];
      }
    }
  } else {  // huffman: bits of every code in the tile
    const int32_t cmin = S.cmin;
    const uint64_t* L = lut + S.lut_off;
    const uint64_t e0 = static_cast<uint64_t>(T.row0) * J.dim;
    const uint32_t ne = T.rows * J.dim;
    for (uint32_t l = threadIdx.x; l < ne; l += blockDim.x) {
      uint32_t r = 0;
      const int32_t c = job_code(J, e0 + l, &r);
      local += lut_entry(L, c, cmin) & 0xFF;
    }
  }
  const unsigned long long tot = block_sum<unsigned long long>(local, s_tmp64);
  if (threadIdx.x == 0) tile_sum[tid] = tot;
}

// ---------------------------------------------------------------------------
// K4: layout, headers, pack table, metadata, failure folding (one CTA)
// ---------------------------------------------------------------------------
struct LayoutArgs {
  uint32_t njobs;
  int layout;
  uint8_t* out;
  uint64_t cap;
  uint64_t* d_offsets;
  uint64_t* d_lengths;
  uint8_t* d_meta;
  uint64_t* d_total;
  uint32_t* call_flags;
  DevError* err;
  int skip;  // match_stats: no layout
};

__device__ void layout_body(const DJob* __restrict__ jobs, JobState* st,
                            const uint64_t* __restrict__ tile_sum, uint64_t* __restrict__ tile_off,
                            const LayoutArgs& a) {
  if (a.skip) return;
  __shared__ unsigned long long s_tmp64[33];
  __shared__ unsigned long long s_first;
  if (threadIdx.x == 0) s_first = ~0ull;
  __syncthreads();
  // failure folding: lowest failing job, its first failure
  for (uint32_t j = threadIdx.x; j < a.njobs; j += blockDim.x) {
    if (st[j].err != ~0ull) atomicMin(&s_first, static_cast<unsigned long long>(j));
  }
  __syncthreads();
  const uint64_t base = a.layout == EMBC_LAYOUT_PACKED ? 4 + 16ull * a.njobs : 0;
  // payload sizes + job-relative tile offsets
  for (uint32_t j = threadIdx.x; j < a.njobs; j += blockDim.x) {
    const DJob& J = jobs[j];
    uint64_t P = 0;
    if (J.codec == EMBC_CODEC_RAW) {
      P = 4 * J.N;
      uint64_t o = 0;
      for (uint32_t t = 0; t < J.ntiles; ++t) {
        tile_off[J.tile0 + t] = o;
        o += 0;
      }
    } else {
      uint64_t o = 0;
      for (uint32_t t = 0; t < J.ntiles; ++t) {
        tile_off[J.tile0 + t] = o;
        o += tile_sum[J.tile0 + t];
      }
      P = J.codec == EMBC_CODEC_VLZ ? o : st[j].payload;
    }
    if (J.N == 0 && J.codec != EMBC_CODEC_HUFFMAN) P = 0;
    st[j].payload = P;
  }
  __syncthreads();
  // chunk offsets: exclusive scan in job order (container.hpp:245-250)
  uint64_t carry = base;
  for (uint32_t j0 = 0; j0 < a.njobs; j0 += blockDim.x) {
    const uint32_t j = j0 + threadIdx.x;
    const uint64_t S = j < a.njobs ? jobs[j].header + st[j].payload : 0;
    unsigned long long tot;
    const unsigned long long pre = block_excl_scan<unsigned long long>(S, s_tmp64, &tot);
    if (j < a.njobs) st[j].chunk_off = carry + pre;
    carry += tot;
  }
  __syncthreads();
  const uint64_t total = carry;
  const bool failed = s_first != ~0ull;
  const bool overflow = !failed && total > a.cap;
  if (threadIdx.x == 0) {
    *a.call_flags = (failed || overflow) ? JF_ABORT : 0;
    if (a.d_total) *a.d_total = (failed || overflow) ? 0 : total;
    if (failed && !a.err->valid) {
      const uint32_t j = static_cast<uint32_t>(s_first);
      const unsigned long long k = st[j].err & ~(1ull << 63);
      a.err->valid = 1;
      a.err->job = j;
      a.err->reason = static_cast<int32_t>(k & 63);
      a.err->index = k >> 6;
      a.err->a = st[j].aux;
      a.err->b = jobs[j].window;
      a.err->eb = jobs[j].qp.eb;
      const int r = a.err->reason;
      a.err->status = (r == EMBC_R_RANGE) ? EMBC_ERR_UNSUPPORTED : EMBC_ERR_VALUE;
    } else if (overflow && !a.err->valid) {
      a.err->valid = 1;
      a.err->job = 0;
      a.err->reason = EMBC_R_CAPACITY;
      a.err->index = 0;
      a.err->a = total;
      a.err->b = a.cap;
      a.err->status = EMBC_ERR_CAPACITY;
    }
  }
  if (failed || overflow) return;
  if (a.layout == EMBC_LAYOUT_PACKED && threadIdx.x == 0) st_le(a.out, a.njobs, 4);
  for (uint32_t j = threadIdx.x; j < a.njobs; j += blockDim.x) {
    const DJob& J = jobs[j];
    const uint64_t off = st[j].chunk_off;
    const uint64_t len = J.header + st[j].payload;
    if (a.d_offsets) a.d_offsets[j] = off;
    if (a.d_lengths) a.d_lengths[j] = len;
    if (a.layout == EMBC_LAYOUT_PACKED) {  // pack table (container.hpp:244-250)
      st_le(a.out + 4 + 16ull * j, off, 8);
      st_le(a.out + 12 + 16ull * j, len, 8);
    }
    uint64_t ebits;
    memcpy(&ebits, &J.qp.eb, 8);
    if (J.header) {  // serialize_chunk header (container.hpp:74-85)
      uint8_t* h = a.out + off;
      h[0] = 'E';
      h[1] = 'M';
      h[2] = 'B';
      h[3] = 'C';
      h[4] = 1;
      h[5] = J.codec;
      st_le(h + 6, ebits, 8);
      st_le(h + 14, J.dim, 4);
      st_le(h + 18, J.n, 4);
      st_le(h + 22, st[j].payload, 8);
    }
    if (a.d_meta) {  // serialize_metadata(metadata_for(chunk)) (container.hpp:196-209)
      uint8_t* m = a.d_meta + static_cast<uint64_t>(kMetaSize) * j;
      st_le(m, kHeader + st[j].payload, 8);
      m[8] = J.codec;
      st_le(m + 9, ebits, 8);
      st_le(m + 17, J.dim, 4);
      st_le(m + 21, J.n, 4);
    }
  }
}

// K3 kernel: vlz decisions / huffman bit counts per tile; the last CTA to
// finish lays the call out (one launch instead of two).
__global__ void __launch_bounds__(kBlock) k_sizes(const DJob* __restrict__ jobs,
                                                  const DTile* __restrict__ tiles,
                                                  const uint32_t* __restrict__ tile_list, uint32_t nlist,
                                                  JobState* __restrict__ st,
                                                  const uint64_t* __restrict__ row_hash,
                                                  const uint32_t* __restrict__ row_lit,
                                                  uint32_t* __restrict__ row_off,
                                                  const uint64_t* __restrict__ lut,
                                                  uint64_t* __restrict__ tile_sum,
                                                  uint64_t* __restrict__ tile_off,
                                                  uint32_t* __restrict__ done_ctr, LayoutArgs la) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_last;
  if (blockIdx.x < nlist)
    sizes_tile(jobs, tiles, tile_list, st, row_hash, row_lit, row_off, lut, tile_sum, smem);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(done_ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    __threadfence();
    layout_body(jobs, st, tile_sum, tile_off, la);
  }
}

// ---------------------------------------------------------------------------
// K5: byte emission
// ---------------------------------------------------------------------------
constexpr uint32_t kStageBytes = 48 * 1024;

__global__ void __launch_bounds__(kBlock) k_emit(const DJob* __restrict__ jobs,
                                                 const DTile* __restrict__ tiles,
                                                 JobState* __restrict__ st,
                                                 const uint32_t* __restrict__ row_off,
                                                 const uint32_t* __restrict__ row_lit,
                                                 const uint64_t* __restrict__ tile_off,
                                                 const uint64_t* __restrict__ tile_sum,
                                                 const uint64_t* __restrict__ lut,
                                                 const uint8_t* __restrict__ books,
                                                 uint64_t book_stride, uint8_t* __restrict__ out,
                                                 uint8_t* __restrict__ edges,
                                                 const uint32_t* __restrict__ call_flags) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t s_tmp32[33];
  __shared__ unsigned long long s_tmp64[33];
  if (*call_flags & JF_ABORT) return;
  const uint32_t tid = blockIdx.x;
  const DTile T = tiles[tid];
  const DJob& J = jobs[T.job];
  JobState& S = st[T.job];
  const uint32_t dim = J.dim;
  const uint64_t e0 = static_cast<uint64_t>(T.row0) * dim;
  const uint32_t ne = T.rows * dim;
  uint8_t* pay = out + S.chunk_off + J.header;

  if (J.codec == EMBC_CODEC_RAW) {  // u32le codes (container.hpp:128-133)
    uint8_t* dst = pay + 4 * e0;
    const uint32_t mis = static_cast<uint32_t>(reinterpret_cast<uint64_t>(dst) & 15);
    for (uint32_t l = threadIdx.x; l < ne; l += blockDim.x) {
      uint32_t r = 0;
      const uint32_t c = static_cast<uint32_t>(job_code(J, e0 + l, &r));
      uint8_t* s = smem + mis + 4 * l;
      s[0] = static_cast<uint8_t>(c);
      s[1] = static_cast<uint8_t>(c >> 8);
      s[2] = static_cast<uint8_t>(c >> 16);
      s[3] = static_cast<uint8_t>(c >> 24);
    }
    __syncthreads();
    copy_out_staged(dst, smem, 4ull * ne);
    return;
  }

  if (J.codec == EMBC_CODEC_VLZ) {  // token stream (vlz.hpp:111-125)
    uint8_t* dst = pay + tile_off[tid];
    const uint32_t mis = static_cast<uint32_t>(reinterpret_cast<uint64_t>(dst) & 15);
    uint32_t* roff = reinterpret_cast<uint32_t*>(smem + kStageBytes);  // per-row byte offset
    // token sizes, thread-contiguous rows
    const uint32_t per = (T.rows + blockDim.x - 1) / blockDim.x;
    const uint32_t r0 = threadIdx.x * per;
    uint32_t sum = 0;
    for (uint32_t r = r0; r < min(r0 + per, T.rows); ++r) {
      const uint64_t g = J.row_base + T.row0 + r;
      const uint32_t o = row_off[g];
      sum += o ? 1 + varint_len(o) : row_lit[g];
    }
    uint32_t tot;
    uint32_t pre = block_excl_scan<uint32_t>(sum, s_tmp32, &tot);
    for (uint32_t r = r0; r < min(r0 + per, T.rows); ++r) {
      const uint64_t g = J.row_base + T.row0 + r;
      const uint32_t o = row_off[g];
      roff[r] = pre;
      if (o) {  // reference token: 0x01, varint(offset)
        uint8_t* p = smem + mis + pre;
        *p++ = 0x01;
        put_varint(p, o);
        pre += 1 + varint_len(o);
      } else {
        pre += row_lit[g];
      }
    }
    __syncthreads();
    // literal tokens: 0x00 then dim zigzag varints, one warp per row
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (uint32_t r = warp; r < T.rows; r += nwarps) {
      const uint64_t g = J.row_base + T.row0 + r;
      if (row_off[g]) continue;
      uint8_t* p = smem + mis + roff[r];
      if (lane == 0) p[0] = 0x00;
      uint32_t carry = 1;
      for (uint32_t j0 = 0; j0 < dim; j0 += 32) {
        const uint32_t j = j0 + lane;
        uint32_t z = 0, len = 0;
        if (j < dim) {
          uint32_t rr = 0;
          z = zigzag(job_code(J, (e0 + static_cast<uint64_t>(r) * dim) + j, &rr));
          len = varint_len(z);
        }
        const uint32_t inc = warp_incl_scan<uint32_t>(len);
        if (j < dim) put_varint(p + carry + inc - len, z);
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    __syncthreads();
    copy_out_staged(dst, smem, tot);
    return;
  }

  // huffman bitstream: MSB-first (bitstream.hpp:32-51)
  {
    const uint64_t bit0 = tile_off[tid];  // bit offset of this tile in the bitstream
    uint8_t* stream = pay + 12 + 5ull * S.nsym;
    uint8_t* dst = stream + (bit0 >> 3);
    const uint32_t mis = static_cast<uint32_t>(reinterpret_cast<uint64_t>(dst) & 15);
    const uint32_t b0 = static_cast<uint32_t>(bit0 & 7);
    // tile 0 of the job also writes the serialized codebook (huffman.hpp:202-209)
    if (T.row0 == 0) {
      const uint8_t* bk = books + static_cast<uint64_t>(J.hjob) * book_stride;
      const uint64_t blen = 12 + 5ull * S.nsym;
      for (uint64_t k = threadIdx.x; k < blen; k += blockDim.x) pay[k] = bk[k];
    }
    int32_t* codes = reinterpret_cast<int32_t*>(smem + kStageBytes);  // padded: l + l/32
    for (uint32_t l = threadIdx.x; l < ne; l += blockDim.x) {
      uint32_t r = 0;
      codes[l + (l >> 5)] = job_code(J, e0 + l, &r);
    }
    uint32_t* words = reinterpret_cast<uint32_t*>(smem);
    const uint32_t nwords = static_cast<uint32_t>((8 * mis + b0 + tile_sum[tid]) >> 5) + 2;
    for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x) words[w] = 0;
    __syncthreads();
    const int32_t cmin = S.cmin;
    const uint64_t* L = lut + S.lut_off;
    const uint32_t per = (ne + blockDim.x - 1) / blockDim.x;
    const uint32_t l0 = threadIdx.x * per, l1 = min(l0 + per, ne);
    uint32_t nb = 0;
    for (uint32_t l = l0; l < l1; ++l) nb += lut_entry(L, codes[l + (l >> 5)], cmin) & 0xFF;
    uint32_t tot;
    uint32_t pos = block_excl_scan<uint32_t>(nb, s_tmp32, &tot) + 8 * mis + b0;
    for (uint32_t l = l0; l < l1; ++l) {
      const uint64_t e = lut_entry(L, codes[l + (l >> 5)], cmin);
      const uint32_t len = static_cast<uint32_t>(e & 0xFF);
      const uint64_t cw = e >> 8;
      const uint32_t off = pos & 31;
      const uint64_t v = cw << (64 - off - len);
      atomicOr(&words[pos >> 5], static_cast<uint32_t>(v >> 32));
      const uint32_t lo = static_cast<uint32_t>(v);
      if (lo) atomicOr(&words[(pos >> 5) + 1], lo);
      pos += len;
    }
    __syncthreads();
    const uint32_t endbit = 8 * mis + b0 + tot;
    const uint32_t nbytes_stage = (endbit + 7) / 8;  // stage bytes incl. the leading `mis`
    for (uint32_t w = threadIdx.x; w < (nbytes_stage + 3) / 4; w += blockDim.x)
      words[w] = __byte_perm(words[w], 0, 0x0123);
    __syncthreads();
    const uint32_t nbytes = nbytes_stage - mis;
    // boundary bytes shared with the neighbouring tiles are merged by K6
    if (threadIdx.x == 0) {
      edges[2 * tid] = smem[mis];                  // first byte (partial if b0 != 0)
      edges[2 * tid + 1] = smem[nbytes_stage - 1];  // last byte (partial if endbit % 8)
    }
    copy_out_staged(dst, smem, nbytes);
    // the job's last tile to finish merges the bytes shared by adjacent tiles
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&S.tiles_done, 1u) == J.ntiles - 1;
    __syncthreads();
    if (s_last) {
      __threadfence();
      for (uint32_t k = 1 + threadIdx.x; k < J.ntiles; k += blockDim.x) {
        const uint32_t t2 = J.tile0 + k;
        const uint64_t b = __ldcg(tile_off + t2);
        if (b & 7) stream[b >> 3] = __ldcg(edges + 2 * (t2 - 1) + 1) | __ldcg(edges + 2 * t2);
      }
    }
  }
}

__global__ void k_count_refs(const uint32_t* __restrict__ row_off, uint32_t n,
                             unsigned long long* __restrict__ cnt) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool ref = i < n && row_off[i] != 0;
  const bool lit = i < n && row_off[i] == 0;
  const uint32_t nr = __popc(__ballot_sync(0xffffffffu, ref));
  const uint32_t nl = __popc(__ballot_sync(0xffffffffu, lit));
  if ((threadIdx.x & 31) == 0) {
    if (nl) atomicAdd(&cnt[0], nl);
    if (nr) atomicAdd(&cnt[1], nr);
  }
}

}  // namespace embc_dev

// ===========================================================================
// host orchestration
// ===========================================================================
namespace embc_host {

using namespace embc_dev;

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
  // target ~2 tiles per SM on a 148-SM part, 1K..8K values per tile
  uint64_t target = total_values / 296;
  target = std::max<uint64_t>(1024, std::min<uint64_t>(8192, target));
  uint32_t rows = static_cast<uint32_t>(std::max<uint64_t>(1, target / std::max<uint32_t>(dim, 1)));
  rows = std::min<uint32_t>(rows, 1024);
  while (rows > 1 && static_cast<uint64_t>(rows) * dim > 8192) --rows;
  if (static_cast<uint64_t>(rows) * dim < 8) rows = std::min<uint32_t>(1024, (8 + dim - 1) / dim);
  return rows;
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

// match_stats (vlz.hpp:162-168): the K1/K3 dedup decisions of one job, counted.
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
  std::vector<DJob> jobs(njobs);
  std::vector<DTile> tiles;
  uint64_t total_values = 0, total_rows = 0;
  for (uint32_t j = 0; j < njobs; ++j) total_values += static_cast<uint64_t>(hj[j].dim) * hj[j].n;
  uint32_t nhuff = 0;
  uint64_t hist_entries = 0;
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
    if (in.dim > 8192)
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
    J.tile_rows = pick_tile_rows(in.dim, total_values);
    J.tile0 = static_cast<uint32_t>(tiles.size());
    for (uint32_t r = 0; r < in.n; r += J.tile_rows) {
      DTile t{};
      t.job = j;
      t.row0 = r;
      t.rows = std::min<uint32_t>(J.tile_rows, in.n - r);
      tiles.push_back(t);
    }
    J.ntiles = static_cast<uint32_t>(tiles.size()) - J.tile0;
  }
  const uint32_t ntiles = static_cast<uint32_t>(tiles.size());
  std::vector<uint32_t> list_nonraw, list_huff_tiles, list_hjobs;
  for (uint32_t t = 0; t < ntiles; ++t) {
    const uint8_t c = jobs[tiles[t].job].codec;
    if (c != EMBC_CODEC_RAW) list_nonraw.push_back(t);
    if (c == EMBC_CODEC_HUFFMAN) list_huff_tiles.push_back(t);
  }
  uint64_t book_cap = 1;
  for (uint32_t j = 0; j < njobs; ++j)
    if (jobs[j].codec == EMBC_CODEC_HUFFMAN) {
      list_hjobs.push_back(j);
      book_cap = std::max<uint64_t>(book_cap, jobs[j].hist_cap);
    }
  uint64_t p2cap = 1;
  while (p2cap < book_cap) p2cap <<= 1;
  const uint64_t book_stride = align_up(12 + 5 * book_cap, 16);
  const bool big_books = p2cap > kSmemBook;

  // ---- scratch carve
  Carve cv;
  const size_t o_jobs = cv.take<DJob>(njobs);
  const size_t o_tiles = cv.take<DTile>(ntiles);
  const size_t o_st = cv.take<JobState>(njobs);
  const size_t o_l1 = cv.take<uint32_t>(list_nonraw.size() + 1);
  const size_t o_l2 = cv.take<uint32_t>(list_huff_tiles.size() + 1);
  const size_t o_l3 = cv.take<uint32_t>(list_hjobs.size() + 1);
  const size_t o_flags = cv.take<uint32_t>(4);
  const size_t host_bytes = cv.off;  // everything above is uploaded from the host
  const size_t o_hash = cv.take<uint64_t>(total_rows + 1);
  const size_t o_lit = cv.take<uint32_t>(total_rows + 1);
  const size_t o_off = cv.take<uint32_t>(total_rows + 1);
  const size_t o_tsum = cv.take<uint64_t>(ntiles + 1);
  const size_t o_toff = cv.take<uint64_t>(ntiles + 1);
  const size_t o_edges = cv.take<uint8_t>(2ull * ntiles + 2);
  hist_entries += kWidePool;  // [nhuff windows | wide pool], LUT mirrors the layout
  const size_t o_lut = cv.take<uint64_t>(hist_entries + 1);
  const size_t o_books = cv.take<uint8_t>(book_stride * std::max<uint32_t>(nhuff, 1));
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
  std::memcpy(hs + o_l1, list_nonraw.data(), sizeof(uint32_t) * list_nonraw.size());
  std::memcpy(hs + o_l2, list_huff_tiles.data(), sizeof(uint32_t) * list_huff_tiles.size());
  std::memcpy(hs + o_l3, list_hjobs.data(), sizeof(uint32_t) * list_hjobs.size());
  std::memset(hs + o_flags, 0, 16);
  uint8_t* d = ctx->d_scratch;
  ce = cudaMemcpyAsync(d, hs, host_bytes, cudaMemcpyHostToDevice, stream);
  if (ce == cudaSuccess) ce = stage_commit(ctx, slot, stream);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "descriptor upload");

  const DJob* d_jobs = reinterpret_cast<const DJob*>(d + o_jobs);
  const DTile* d_tiles = reinterpret_cast<const DTile*>(d + o_tiles);
  JobState* d_st = reinterpret_cast<JobState*>(d + o_st);
  uint32_t* d_flags = reinterpret_cast<uint32_t*>(d + o_flags);
  uint64_t* d_hash = reinterpret_cast<uint64_t*>(d + o_hash);
  uint32_t* d_lit = reinterpret_cast<uint32_t*>(d + o_lit);
  uint32_t* d_off = reinterpret_cast<uint32_t*>(d + o_off);
  uint64_t* d_tsum = reinterpret_cast<uint64_t*>(d + o_tsum);
  uint64_t* d_toff = reinterpret_cast<uint64_t*>(d + o_toff);
  uint8_t* d_edges = d + o_edges;
  uint64_t* d_lut = reinterpret_cast<uint64_t*>(d + o_lut);
  uint8_t* d_books = d + o_books;
  uint32_t* d_hist = reinterpret_cast<uint32_t*>(ctx->d_hist);

  // The staged job state makes a raw-only call with a bad window impossible;
  // the stage-2 key above is folded like any other device failure.
  const uint32_t max_rows_stride = [&] {
    uint32_t m = 0;
    for (uint32_t j = 0; j < njobs; ++j) m = std::max(m, jobs[j].tile_rows * (jobs[j].dim | 1u));
    return m;
  }();
  const uint32_t hist_smem_off = static_cast<uint32_t>(align_up(sizeof(int32_t) * max_rows_stride, 16));
  if (ntiles) {
    EMBC_TIMED(ctx, "k_quant_stats", stream,
               k_quant_stats<<<ntiles, kBlock, hist_smem_off + (nhuff ? sizeof(uint32_t) * kWin : 0), stream>>>(
                   d_jobs, d_tiles, d_st, d_hash, d_lit, d_hist, hist_smem_off));
  }
  if (!list_hjobs.empty()) {
    BookScratch gs{};
    if (big_books) {
      gs.key = reinterpret_cast<uint64_t*>(d + o_gkey);
      gs.wgt = reinterpret_cast<uint64_t*>(d + o_gwgt);
      gs.parent = reinterpret_cast<int32_t*>(d + o_gpar);
    }
    const size_t sm = kSmemBook * (8 + 16 + 8);
    EMBC_TIMED(ctx, "k_huff_book", stream,
               k_huff_book<<<static_cast<uint32_t>(list_hjobs.size()), kBookThreads, sm, stream>>>(
                   d_jobs, reinterpret_cast<const uint32_t*>(d + o_l3), d_st, d_hist, d_lut, d_books,
                   book_stride, gs, p2cap, nhuff, reinterpret_cast<unsigned long long*>(d_flags + 2)));
  }
  LayoutArgs la{};
  la.njobs = njobs;
  la.layout = layout;
  la.out = d_out;
  la.cap = cap;
  la.d_offsets = d_offsets;
  la.d_lengths = d_lengths;
  la.d_meta = d_meta;
  la.d_total = d_total;
  la.call_flags = d_flags;
  la.err = ctx->d_err;
  la.skip = d_stats ? 1 : 0;
  {
    const uint32_t nl = static_cast<uint32_t>(list_nonraw.size());
    EMBC_TIMED(ctx, "k_sizes", stream,
               k_sizes<<<nl + 1, kBlock, sizeof(uint64_t) * kHashStage, stream>>>(
                   d_jobs, d_tiles, reinterpret_cast<const uint32_t*>(d + o_l1), nl, d_st, d_hash, d_lit, d_off,
                   d_lut, d_tsum, d_toff, d_flags + 1, la));
  }
  if (d_stats) {  // match_stats: count literal vs reference rows of job 0
    k_count_refs<<<(static_cast<uint32_t>(total_rows) + 255) / 256, 256, 0, stream>>>(
        d_off, static_cast<uint32_t>(total_rows), d_stats);
    ce = cudaGetLastError();
    return ce == cudaSuccess ? EMBC_OK : cuda_fail(ctx, ce, "match_stats launch");
  }
  if (ntiles) {
    EMBC_TIMED(ctx, "k_emit", stream,
               k_emit<<<ntiles, kBlock, kStageBytes + 36 * 1024, stream>>>(
                   d_jobs, d_tiles, d_st, d_off, d_lit, d_toff, d_tsum, d_lut, d_books, book_stride, d_out,
                   d_edges, d_flags));
  }
  ce = cudaGetLastError();
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "encode launch");
  return EMBC_OK;
}

cudaError_t encode_set_attributes() {
  cudaError_t e = cudaFuncSetAttribute(k_emit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kStageBytes + 36 * 1024);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_huff_book, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kSmemBook * (8 + 16 + 8));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_quant_stats, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           sizeof(int32_t) * 16384 * 2 + sizeof(uint32_t) * kWin);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_sizes, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              sizeof(uint64_t) * kHashStage);
}

}  // namespace embc_host
