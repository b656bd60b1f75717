// encode_timeline.cuh -- EMBC_DEBUG builds only (make EXTRA=-DEMBC_DEBUG):
// per-phase %globaltimer stamps of the encode kernels and the reports that
// print them (tools/gpu_iter.sh).  Product builds see empty macros.
#pragma once
#ifdef EMBC_DEBUG
__device__ unsigned long long g_dbg[8];
__device__ unsigned long long g_ts[16384][10];
__device__ uint32_t g_tc[16384];  // codec of the tile
__device__ unsigned long long g_kspan[4] = {~0ull, 0, 0, 0};  // k_encode: first CTA start, last CTA end, CTAs done, calls
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TS(k) do { if (threadIdx.x == 0 && tid < 16384) g_ts[tid][k] = gtime(); } while (0)
// E2 (fused phase) timeline: every CTA stamps its exit; the last one prints
// per-phase means / maxima (0 start, 1 codes, 2 sizes, 3 look-back, 4 staged, 5 exit)
struct EmitEnd {
  uint32_t tid, n;
  __device__ ~EmitEnd() {
    if (threadIdx.x != 0 || tid >= 16384 || n == 0xFFFFFFFFu) return;
    g_ts[tid][5] = gtime();
    __threadfence();
    if (atomicAdd(&g_dbg[4], 1ull) != n - 1) return;
    g_dbg[4] = 0;
    if (n < 100 || (atomicAdd(&g_dbg[5], 1ull) % 8) != 7) return;
    unsigned long long t0 = ~0ull, t1 = 0, sm[6] = {0}, mx[6] = {0};
    for (uint32_t t = 0; t < n && t < 16384; ++t) {
      t0 = min(t0, g_ts[t][0]);
      t1 = max(t1, g_ts[t][5]);
    }
    for (uint32_t t = 0; t < n && t < 16384; ++t) {
      unsigned long long prev = g_ts[t][0];
      sm[0] += prev - t0;
      mx[0] = max(mx[0], prev - t0);
      for (int k = 1; k < 6; ++k) {
        if (g_ts[t][k] < prev) continue;
        const unsigned long long d = g_ts[t][k] - prev;
        sm[k] += d;
        mx[k] = max(mx[k], d);
        prev = g_ts[t][k];
      }
    }
    for (uint32_t cd = 0; cd < 3; ++cd) {  // codes + sizes by codec
      unsigned long long c1 = 0, m1 = 0, c2 = 0, m2 = 0, nn = 0;
      for (uint32_t t = 0; t < n && t < 16384; ++t) {
        if (g_tc[t] != cd || g_ts[t][2] < g_ts[t][1] || g_ts[t][1] < g_ts[t][0]) continue;
        ++nn;
        c1 += g_ts[t][1] - g_ts[t][0];
        m1 = max(m1, g_ts[t][1] - g_ts[t][0]);
        c2 += g_ts[t][2] - g_ts[t][1];
        m2 = max(m2, g_ts[t][2] - g_ts[t][1]);
      }
      if (nn) printf("  codec %u: %llu tiles codes %llu/%llu sizes %llu/%llu\n", cd, nn, c1 / nn, m1, c2 / nn, m2);
      if (cd == 1 && nn) {
        unsigned long long a6 = 0, a7 = 0, a8 = 0, m6 = 0, m7 = 0, m8 = 0, rr = 0, mr = 0;
        for (uint32_t t = 0; t < n && t < 16384; ++t) {
          if (g_tc[t] != 1 || !g_ts[t][6] || !g_ts[t][8]) continue;
          a6 += g_ts[t][6] - g_ts[t][1]; m6 = max(m6, g_ts[t][6] - g_ts[t][1]);
          a7 += g_ts[t][7] - g_ts[t][6]; m7 = max(m7, g_ts[t][7] - g_ts[t][6]);
          a8 += g_ts[t][8] - g_ts[t][7]; m8 = max(m8, g_ts[t][8] - g_ts[t][7]);
          rr += g_ts[t][9]; mr = max(mr, g_ts[t][9]);
          g_ts[t][6] = g_ts[t][8] = 0;
        }
        printf("  vlz sizes: stage %llu/%llu search %llu/%llu verify %llu/%llu rounds %llu/%llu\n", a6 / nn, m6, a7 / nn,
               m7, a8 / nn, m8, rr / nn, mr);
      }
    }
    printf("k_emit: %u tiles span %llu ns; start %llu/%llu codes %llu/%llu sizes %llu/%llu lookback %llu/%llu bytes %llu/%llu exit %llu/%llu\n",
           n, t1 - t0, sm[0] / n, mx[0], sm[1] / n, mx[1], sm[2] / n, mx[2], sm[3] / n, mx[3], sm[4] / n, mx[4],
           sm[5] / n, mx[5]);
    for (uint32_t t = 0; t < n && t < 16384; ++t)
      for (int k = 0; k < 10; ++k) g_ts[t][k] = 0;
  }
};
__device__ unsigned long long g_ts1[16384][14];
#define TS1(k) do { if (threadIdx.x == 0 && blockIdx.x < 16384) g_ts1[blockIdx.x][k] = gtime(); } while (0)
#define TS1V(k, v) do { if (threadIdx.x == 0 && blockIdx.x < 16384) g_ts1[blockIdx.x][k] = (v); } while (0)
template <class A>
__device__ void dbg_stats_report(const A& a) {
  if (threadIdx.x == 0 && atomicAdd(&g_dbg[2], 1ull) == a.ntiles - 1 && (g_dbg[2] = 0, a.ntiles > 100) &&
      atomicAdd(&g_dbg[3], 1ull) % 8 == 7) {
    unsigned long long t0 = ~0ull, mxe = 0, sl = 0, ml = 0, sb = 0, mb = 0, nb = 0;
    for (uint32_t t = 0; t < a.ntiles; ++t) t0 = min(t0, g_ts1[t][0]);
    for (uint32_t t = 0; t < a.ntiles; ++t) {
      mxe = max(mxe, g_ts1[t][4] - t0);
      sl += g_ts1[t][1] - g_ts1[t][0];
      ml = max(ml, g_ts1[t][1] - g_ts1[t][0]);
      if (g_ts1[t][4] != g_ts1[t][3]) {
        ++nb;
        sb += g_ts1[t][4] - g_ts1[t][3];
        mb = max(mb, g_ts1[t][4] - g_ts1[t][3]);
      }
    }
    printf("k_stats: span %llu ns, tile main mean %llu max %llu, books %llu mean %llu max %llu ns\n", mxe,
           sl / a.ntiles, ml, nb, nb ? sb / nb : 0, mb);
    for (uint32_t t = 0; t < a.ntiles; ++t) {
      if (g_ts1[t][4] - g_ts1[t][3] != mb) continue;
      const unsigned long long* g = g_ts1[t];
      printf("  slowest book: S %llu count %llu compact %llu sort %llu merge %llu depth %llu csort %llu rest %llu"
             " (nsym %llu span %llu)\n",
             g[5] - g[3], g[6] - g[5], g[7] - g[6], g[8] - g[7], g[9] - g[8], g[10] - g[9], g[11] - g[10], g[4] - g[11],
             g[12], g[13]);
    }
    // book time by alphabet size
    unsigned long long cnt[6] = {0}, tot[6] = {0}, mxb[6] = {0};
    for (uint32_t t = 0; t < a.ntiles; ++t) {
      if (g_ts1[t][4] == g_ts1[t][3]) continue;
      const unsigned long long ns = g_ts1[t][12], d = g_ts1[t][4] - g_ts1[t][3];
      const int b = ns <= 8 ? 0 : ns <= 32 ? 1 : ns <= 64 ? 2 : ns <= 128 ? 3 : ns <= 256 ? 4 : 5;
      ++cnt[b]; tot[b] += d; mxb[b] = max(mxb[b], d);
    }
    printf("  books by nsym (<=8,<=32,<=64,<=128,<=256,more): n/mean/max");
    for (int b = 0; b < 6; ++b) printf(" %llu/%llu/%llu", cnt[b], cnt[b] ? tot[b] / cnt[b] : 0, mxb[b]);
    printf("\n");
  }
}
__device__ __forceinline__ void dbg_kspan_begin() {
  if (threadIdx.x == 0) atomicMin(&g_kspan[0], gtime());
}
__device__ __forceinline__ void dbg_kspan_end(uint32_t ntiles) {
  if (threadIdx.x != 0) return;
  atomicMax(&g_kspan[1], gtime());
  __threadfence();
  if (atomicAdd(&g_kspan[2], 1ull) == ntiles - 1) {
    const unsigned long long k = atomicAdd(&g_kspan[3], 1ull);
    if (k < 400) printf("KSPAN enc %llu %llu\n", g_kspan[0], atomicMax(&g_kspan[1], 0ull));
    g_kspan[0] = ~0ull;
    g_kspan[1] = 0;
    g_kspan[2] = 0;
  }
}
#define EMBC_DBG(...) __VA_ARGS__
#else
#define EMBC_DBG(...) do {} while (0)
#define TS(k) do {} while (0)
#define TS1(k) do {} while (0)
#define TS1V(k, v) do {} while (0)
#endif
