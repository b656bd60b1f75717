// decode_timeline.cuh -- EMBC_DEBUG builds only (make EXTRA=-DEMBC_DEBUG):
// per-role %globaltimer stamps of k_dec_main and the report that prints them
// (tools/gpu_iter.sh).  Product builds see empty macros.
#pragma once
#ifdef EMBC_DEBUG
__device__ unsigned long long g_dts[16384][12];  // role, t1..t11 (t7 = end)
__device__ unsigned long long g_cta0[16384];     // %globaltimer at each CTA's first instruction
__device__ unsigned long long g_dcalls;
__device__ unsigned long long g_kspan[4] = {~0ull, 0, 0, 0};  // k_dec_main: first start, last end, CTAs done, calls
__device__ unsigned long long g_dloc[12];  // huffman blocks: local tables ok / not; ns in local build, in stage, ...
__device__ __forceinline__ unsigned long long dtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define DTS(slot, k) do { if (threadIdx.x == 0 && (slot) < 16384) g_dts[slot][k] = dtime(); } while (0)
#define DROLE(slot, r) do { if (threadIdx.x == 0 && (slot) < 16384) { g_dts[slot][0] = (r); for (int q = 2; q < 12; ++q) g_dts[slot][q] = 0; } } while (0)
template <class A>
__device__ void dbg_decode_report(const A& a) {
    if (threadIdx.x != 0) return;
    const uint32_t nb = a.nchunks + a.nseg + a.nhblk + a.nraw + a.nctile + a.nchunks - 1;
    if ((++g_dcalls) % 8 == 7 && nb <= 16384) {
      printf("D1 huffman blocks: local tables %llu, waited %llu; mean ns local build %llu (warp %llu, lut %llu), stage %llu\n",
             g_dloc[0], g_dloc[1], g_dloc[2] / max(1ull, g_dloc[0] + g_dloc[1]), g_dloc[4] / max(1ull, g_dloc[0]),
             g_dloc[5] / max(1ull, g_dloc[0]), g_dloc[3] / max(1ull, g_dloc[0] + g_dloc[1]));
      for (int q = 0; q < 12; ++q) g_dloc[q] = 0;
      unsigned long long t0 = ~0ull;
      for (uint32_t k = 0; k < nb; ++k) t0 = min(t0, g_dts[k][1]);
      const char* names[6] = {"chunk", "vlzseg", "hufblk", "raw", "copy", "finish"};
      {  // CTA dispatch: first instruction of every CTA relative to the earliest role stamp
        unsigned long long c0 = ~0ull, c1 = 0, cl = 0, cend = 0;
        for (uint32_t k = 0; k < nb; ++k) {
          c0 = min(c0, g_cta0[k]);
          c1 = max(c1, g_cta0[k]);
          cend = max(cend, g_dts[k][7]);
        }
        cl = g_cta0[nb - 1];
        printf("D1 cta starts: first %lld last %lld (last block %lld) last role end %lld ns (rel. to first role stamp)\n",
               (long long)(c0 - t0), (long long)(c1 - t0), (long long)(cl - t0), (long long)(cend - t0));
      }
      {  // huffman table build phases (slots 8000 + chunk: 8 start, 2 keys, 3 sort, 4 codes, 5 lut, 6 dup sort)
        unsigned long long n = 0, sm[6] = {0}, mx[6] = {0};
        const int ord[6] = {8, 2, 3, 4, 5, 6};
        for (uint32_t c = 0; c < a.nchunks && 8000 + c < 16384; ++c) {
          if (!g_dts[8000 + c][8] || !g_dts[8000 + c][6]) continue;
          ++n;
          for (int q = 1; q < 6; ++q) {
            const unsigned long long d = g_dts[8000 + c][ord[q]] - g_dts[8000 + c][ord[q - 1]];
            sm[q] += d;
            mx[q] = max(mx[q], d);
          }
          sm[0] += g_dts[8000 + c][8] - t0;
          mx[0] = max(mx[0], g_dts[8000 + c][8] - t0);
        }
        if (n)
          printf("D1 tables n %llu start %llu/%llu keys %llu/%llu sort %llu/%llu codes %llu/%llu lut %llu/%llu dup %llu/%llu\n", n,
                 sm[0] / n, mx[0], sm[1] / n, mx[1], sm[2] / n, mx[2], sm[3] / n, mx[3], sm[4] / n, mx[4], sm[5] / n, mx[5]);
        for (uint32_t c = 0; c < a.nchunks && 8000 + c < 16384; ++c) g_dts[8000 + c][8] = g_dts[8000 + c][6] = 0;
      }
      for (uint32_t role = 0; role < 6; ++role) {
        unsigned long long n = 0, mn = ~0ull, mx = 0, sum[12] = {0}, mxs[12] = {0};
        for (uint32_t k = 0; k < nb; ++k) {
          if (g_dts[k][0] != role) continue;
          ++n;
          mn = min(mn, g_dts[k][1] - t0);
          mx = max(mx, g_dts[k][7] - t0);
          unsigned long long prev = g_dts[k][1];
          for (int q = 2; q <= 7; ++q) {
            if (!g_dts[k][q]) continue;
            if (q == 7 && g_dts[k][8]) {  // extra stamps 8..11 recorded between 6 and 7
              for (int x = 8; x <= 11; ++x) {
                if (!g_dts[k][x]) continue;
                const unsigned long long d = g_dts[k][x] - prev;
                sum[x] += d;
                mxs[x] = max(mxs[x], d);
                prev = g_dts[k][x];
              }
            }
            const unsigned long long d = g_dts[k][q] - prev;
            sum[q] += d;
            mxs[q] = max(mxs[q], d);
            prev = g_dts[k][q];
          }
        }
        if (!n) continue;
        printf("D1 %-6s n %4llu span [%6llu %6llu] phase mean/max ns: 2:%llu/%llu 3:%llu/%llu 4:%llu/%llu 5:%llu/%llu 6:%llu/%llu 8:%llu/%llu 9:%llu/%llu 10:%llu/%llu 11:%llu/%llu 7:%llu/%llu\n",
               names[role], n, mn, mx, sum[2] / n, mxs[2], sum[3] / n, mxs[3], sum[4] / n, mxs[4], sum[5] / n, mxs[5],
               sum[6] / n, mxs[6], sum[8] / n, mxs[8], sum[9] / n, mxs[9], sum[10] / n, mxs[10], sum[11] / n, mxs[11], sum[7] / n, mxs[7]);
      }
    }
}
#define EMBC_DBG(...) __VA_ARGS__
#else
#define EMBC_DBG(...) do {} while (0)
#define DTS(slot, k) do {} while (0)
#define DROLE(slot, r) do {} while (0)
#endif
