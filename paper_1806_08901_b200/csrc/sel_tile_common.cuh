// sel_tile_common.cuh -- shared pieces of the TMA tile pipeline kernels (k_tile in
// sel_tile.cu: one field per launch; k_batch in sel_batch.cu: a whole batch per launch).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "sel_device.cuh"

namespace sel {


// tile configuration (developer overrides for sweeps: -DSEL_CW2=... etc.)
#ifndef SEL_CW2
#define SEL_CW2 24
#endif
#ifndef SEL_STAGES2
#define SEL_STAGES2 3
#endif
#ifndef SEL_TB2
#define SEL_TB2 8192
#endif
#ifndef SEL_CW3
#define SEL_CW3 8
#endif
#ifndef SEL_STAGES3
#define SEL_STAGES3 2
#endif
#ifndef SEL_TB3
#define SEL_TB3 8704
#endif

constexpr int kBoxK = 4 * 32 + 4;             // 132 floats: 4 halo columns (last one used) + 128
constexpr int kHBins = 1024;                  // histogram window: codes [-512, 512)
constexpr int kHStride = kHBins + 1;          // copy stride (words): copy c of a bin -> bank + c
constexpr uint32_t kHOff = kSlotOff + (uint32_t)(kCenter - kHBins / 2);

template <int D>
struct TileCfg {
  static constexpr int CW = D == 3 ? SEL_CW3 : SEL_CW2;           // consumer warps
  static constexpr int THREADS = (CW + 1) * 32;
  static constexpr int BOXJ = 4 * CW + 1;                         // halo row + 4 per warp
  static constexpr int BOXI = D == 3 ? 5 : 1;                     // halo plane + 4 (3D)
  static constexpr int PLANE = kBoxK * BOXJ;                      // floats per smem plane
  static constexpr uint32_t STAGE_BYTES = PLANE * BOXI * 4;
  static constexpr int STAGE_FLOATS = ((STAGE_BYTES + 127) & ~127) / 4;
  static constexpr int STAGES = D == 3 ? SEL_STAGES3 : SEL_STAGES2;
  static constexpr int COPIES = D == 3 ? 4 : 8;                   // histogram lane copies
  static constexpr int HIST_WORDS = (COPIES + 1) * kHStride;   // + trash copy
  // second level: one table of TB 32-bit counters centred on code 0 for the codes
  // outside the lane-copy window (wide distributions: noise, fronts, coarse data)
  static constexpr int TB = D == 3 ? SEL_TB3 : SEL_TB2;
  static constexpr int TBL_WORDS = TB;
  static constexpr uint32_t kTOff = kSlotOff + (uint32_t)(kCenter - TB / 2);   // bits -> table slot
  static constexpr size_t SMEM = 128 + (size_t)STAGES * STAGE_FLOATS * 4 + HIST_WORDS * 4 +
                                 TBL_WORDS * 4 + STAGES * 48 + 16;
};

// ------------------------------------------------------------ mbarrier / TMA PTX
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// non-blocking probe of a phase (producers poll it with a sleep: a suspended try_wait
// wakes on every barrier event of the CTA and would steal issue slots from consumers)
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
  while (!mbar_test(bar, parity)) __nanosleep(64);
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            int c2, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
template <int N>
__device__ __forceinline__ void consumer_sync() {   // the consumer threads only
  asm volatile("bar.sync 1, %0;" ::"n"(N) : "memory");
}

// One plane of a warp's tile rows: the 5 smem rows (halo row + 4) of the lane's block
// columns, each with its left neighbour (lane-1's last value; lane 0 reads the halo
// column, which TMA zero-filled at the field's left edge).  All loads are issued first.
__device__ __forceinline__ void load_plane(const float *prow, int lane, float (&v)[5][4],
                                           float (&h)[5]) {
  float h0[5];
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const float4 q = *reinterpret_cast<const float4 *>(prow + r * kBoxK + 4 + 4 * lane);
    v[r][0] = q.x; v[r][1] = q.y; v[r][2] = q.z; v[r][3] = q.w;
    h0[r] = prow[r * kBoxK + 3];
  }
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const float hs = __shfl_up_sync(0xffffffffu, v[r][3], 1);
    h[r] = lane == 0 ? h0[r] : hs;
  }
}

// SZ code of one residual: b = bits(q + M) (reading R5, see sel_device.cuh), w = its
// offset in the window; one unconditional increment of the lane's copy (no divergence):
// out-of-window values land in the copy's pad word (index kHBins), ignored at the flush.
__device__ __forceinline__ uint32_t sz_win(float d, float r_f, unsigned int *hcopy) {
  const uint32_t b = __float_as_uint(__fadd_rn(__fmul_rn(d, r_f), kMagic));
  const uint32_t w = b - kHOff;
  atomicAdd(hcopy + min(w, (uint32_t)kHBins), 1u);
  return w;
}


// Consumer work of one tile task (block-layer bi, tile row btj, tile column btk; warp-level:
// every consumer warp of the CTA calls it for the same tile).  S: the tile's smem stage.  Adds the SZ codes to the CTA's histogram
// (lane copies / packed table / ghist / ovf) and returns the lane's block bits/error.
template <int D, bool DBG>
__device__ __forceinline__ void tile_consume(const float *S, int btk, int btj, int bi,
                                             const TileGeo &tg, int warp,
                                             int lane, bool ok, float r_f, int minexp,
                                             unsigned int *hlane, unsigned int *htrash,
                                             unsigned int *tbl, int *tbl_used, int tbl_mark,
                                             unsigned long long *ghist,
                                             unsigned int &ovf, const DebugPtrs &dbg,
                                             uint64_t &tbits, double &terr) {
  using Cfg = TileCfg<D>;
  constexpr int CW = Cfg::CW;
  constexpr int SZ = Tab<D>::SIZE;
  constexpr int NPL = D == 3 ? 4 : 1;
  // per-axis extents and block coordinates fit 32 bits (tile_supported); only the debug
  // dumps form 64-bit linear indices
  const int n0 = (int)tg.n[0], n1 = (int)tg.n[1], n2 = (int)tg.n[2];
    const int bj = btj * CW + warp;
    const int bk = btk * 32 + lane;
    tbits = 0;
    terr = 0.0;
    if (ok && bj < tg.nb[1]) {
      const bool activeK = bk < tg.nb[2];
      const int I0 = 4 * bi, J0 = 4 * bj, K0 = 4 * bk;
      const float *wrow = S + (4 * warp) * kBoxK;   // smem row of j = J0 - 1 (plane 0)
      unsigned int *const hcopy = activeK ? hlane : htrash;
      // ---------------- SZ: nested differences on the tile (R4), codes -> histogram (R5)
      float dprev[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) dprev[r][c] = 0.0f;
      if constexpr (D == 3) {     // plane i = I0 - 1 (smem plane 0; zeros at i < 0)
        float v[5][4], h[5], d1up[4];
        load_plane(wrow, lane, v, h);
#pragma unroll
        for (int c = 0; c < 4; ++c) d1up[c] = v[0][c] - (c ? v[0][c - 1] : h[0]);
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float d1 = v[r + 1][c] - (c ? v[r + 1][c - 1] : h[r + 1]);
            dprev[r][c] = d1 - d1up[c];
            d1up[c] = d1;
          }
      }
      float blk2[D == 2 ? 16 : 1];   // 2D: the ZFP block is rows 1..4 of the SZ plane
#pragma unroll 1
      for (int p = 0; p < NPL; ++p) {
        const int i = I0 + p;
        float v[5][4], h[5], d1up[4];
        load_plane(wrow + (D == 3 ? (p + 1) * Cfg::PLANE : 0), lane, v, h);
        if constexpr (D == 2) {       // rows past the field's edge replicate the last (R17)
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c)
              blk2[4 * r + c] = (r == 0 || J0 + r < n1) ? v[r + 1][c] : blk2[4 * (r - 1) + c];
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) d1up[c] = v[0][c] - (c ? v[0][c - 1] : h[0]);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int j = J0 + r;
          if (i >= n0 || j >= n1) break;              // padded rows/planes: no SZ point
          uint32_t w[4];
          uint32_t any = 0;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float d1 = v[r + 1][c] - (c ? v[r + 1][c - 1] : h[r + 1]);
            const float d2 = d1 - d1up[c];
            d1up[c] = d1;
            float d;
            if constexpr (D == 3) {
              d = d2 - dprev[r][c];
              dprev[r][c] = d2;
            } else {
              d = d2;
            }
            w[c] = sz_win(d, r_f, hcopy);
            any |= w[c];
          }
          // the field origin is stored verbatim, not coded (R4): undo its count
          const bool orow = (i == 0) && (j == 0) && (btk == 0);
          if (orow && lane == 0) {
            if (w[0] < (uint32_t)kHBins) atomicSub(hcopy + w[0], 1u);
            w[0] = 0u;
          }
          if constexpr (DBG) {
            if (activeK) {
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                if (orow && lane == 0 && c == 0) continue;
                const uint32_t sl = w[c] + (kHOff - kSlotOff);
                dbg.codes[((int64_t)i * n1 + j) * n2 + K0 + c] = sl > 65534u ? kOvfSlot : (int32_t)sl;
              }
            }
          }
          // out-of-window codes (wide distributions): one warp-uniform branch per row; the
          // table takes them with one predicated atomic each, the rest (rare) go to the
          // global histogram or the overflow count
          if (__any_sync(0xffffffffu, activeK && any >= (uint32_t)kHBins)) {
            uint32_t far = 0u;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const uint32_t tb = w[c] + (kHOff - Cfg::kTOff);
              const bool out = activeK && w[c] >= (uint32_t)kHBins;
              if (out && tb < (uint32_t)Cfg::TB) atomicAdd(tbl + tb, 1u);
              far |= (out && tb >= (uint32_t)Cfg::TB) ? (1u << c) : 0u;
            }
            if (lane == 0) *tbl_used = tbl_mark;
            if (__any_sync(0xffffffffu, far != 0u)) {
#pragma unroll
              for (int c = 0; c < 4; ++c)
                if (far & (1u << c)) {
                  const uint32_t sl = w[c] + (kHOff - kSlotOff);
                  if (sl > 65534u) ++ovf;
                  else atomicAdd(ghist + sl, 1ull);
                }
            }
          }
        }
      }
      // ---------------- ZFP on the lane's block, edge-replicated at the far edges (R17)
      if (activeK) {
        float blk[SZ];
        if constexpr (D == 2) {
#pragma unroll
          for (int n = 0; n < 16; ++n) blk[n] = blk2[n];
        } else {
#pragma unroll
          for (int p = 0; p < NPL; ++p) {
            const int ic = min(I0 + p, n0 - 1) - I0;          // 0..3, edge-replicated
            const float *pbase = S + (ic + 1) * Cfg::PLANE;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const int jc = min(J0 + r, n1 - 1) - J0;         // 0..3
              const float4 q = *reinterpret_cast<const float4 *>(
                  pbase + (4 * warp + 1 + jc) * kBoxK + 4 + 4 * lane);
              const int o = (p * 4 + r) * 4;
              blk[o] = q.x; blk[o + 1] = q.y; blk[o + 2] = q.z; blk[o + 3] = q.w;
            }
          }
        }
        uint32_t bits;
        double E;
        int emax;
        int cf[SZ];
        uint32_t u[SZ];
        zfp_block<D, DBG>(blk, minexp, bits, E, emax, cf, u);
        tbits = bits;
        terr = E;
        if constexpr (DBG) {
          const int64_t tb = (D == 3 ? ((int64_t)bi * tg.nb[1] + bj) : (int64_t)bj) * tg.nb[2] + bk;   // block index
          dbg.emax[tb] = emax; dbg.bits[tb] = bits; dbg.err[tb] = E;
#pragma unroll
          for (int n = 0; n < SZ; ++n) { dbg.coef[tb * SZ + n] = cf[n]; dbg.uword[tb * SZ + n] = u[n]; }
        }
      }
    }
}

// Sampled-block task (strides > 1; k_batch): lane = processed block t (act: t < n_pb),
// read with its halo from global memory (L2: the range pass just streamed the field),
// codes into the same smem histogram as a tile task, ZFP block in registers.  Every lane
// of the warp runs (inactive lanes on a clamped block, contributing nothing) so the
// warp-uniform out-of-window branch stays uniform.
template <int D>
__device__ __forceinline__ void sampled_consume(const float *__restrict__ x, const Geo &g,
                                                int64_t t, bool act, float r_f, int minexp,
                                                unsigned int *hlane, unsigned int *htrash,
                                                unsigned int *tbl, int *tbl_used, int tbl_mark,
                                                unsigned long long *ghist, unsigned int &ovf,
                                                uint64_t &tbits, double &terr) {
  using Cfg = TileCfg<D>;
  constexpr int SZ = Tab<D>::SIZE;
  constexpr int PL = D == 3 ? 4 : 1;
  const int lane = threadIdx.x & 31;
  if (!act) t = 0;
  const int64_t p2 = t % g.npb[2];
  const int64_t qq = t / g.npb[2];
  const int64_t p1 = qq % g.npb[1];
  const int64_t p0 = qq / g.npb[1];
  const int64_t I0 = 4 * p0 * g.s[0], J0 = 4 * p1 * g.s[1], K0 = 4 * p2 * g.s[2];
  float blk[SZ];
  float dprev[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) dprev[r][c] = 0.0f;
  if (D == 3 && I0 > 0) {        // plane i = I0 - 1 (zeros outside the field)
    float up[4] = {0.f, 0.f, 0.f, 0.f}, uh = 0.0f;
    if (J0 > 0) load_row<true>(x, g, I0 - 1, J0 - 1, K0, up, uh);
    float d1up[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) d1up[c] = up[c] - (c ? up[c - 1] : uh);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      float v[4], h;
      load_row<true>(x, g, I0 - 1, J0 + r, K0, v, h);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float d1 = v[c] - (c ? v[c - 1] : h);
        dprev[r][c] = d1 - d1up[c];
        d1up[c] = d1;
      }
    }
  }
#pragma unroll
  for (int p = 0; p < PL; ++p) {
    const int64_t i = I0 + p;
    float d1up[4];
    {
      float up[4] = {0.f, 0.f, 0.f, 0.f}, uh = 0.0f;
      if (J0 > 0) load_row<true>(x, g, i, J0 - 1, K0, up, uh);
#pragma unroll
      for (int c = 0; c < 4; ++c) d1up[c] = up[c] - (c ? up[c - 1] : uh);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t j = J0 + r;
      const bool rowok = act && i < g.n[0] && j < g.n[1];   // k < n[2]: n[2] % 4 == 0
      float v[4], h;
      load_row<true>(x, g, i, j, K0, v, h);
      uint32_t w[4];
      uint32_t any = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        blk[(p * 4 + r) * 4 + c] = v[c];
        const float d1 = v[c] - (c ? v[c - 1] : h);
        const float d2 = d1 - d1up[c];
        d1up[c] = d1;
        float d;
        if constexpr (D == 3) {
          d = d2 - dprev[r][c];
          dprev[r][c] = d2;
        } else {
          d = d2;
        }
        const bool valid = rowok && !(i == 0 && j == 0 && K0 + c == 0);   // origin (R4)
        w[c] = sz_win(d, r_f, valid ? hlane : htrash);
        w[c] = valid ? w[c] : 0u;
        any |= w[c];
      }
      if (__any_sync(0xffffffffu, any >= (uint32_t)kHBins)) {
        uint32_t far = 0u;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t tb = w[c] + (kHOff - Cfg::kTOff);
          const bool out = w[c] >= (uint32_t)kHBins;
          if (out && tb < (uint32_t)Cfg::TB) atomicAdd(tbl + tb, 1u);
          far |= (out && tb >= (uint32_t)Cfg::TB) ? (1u << c) : 0u;
        }
        if (lane == 0) *tbl_used = tbl_mark;
        if (__any_sync(0xffffffffu, far != 0u)) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (far & (1u << c)) {
              const uint32_t sl = w[c] + (kHOff - kSlotOff);
              if (sl > 65534u) ++ovf;
              else atomicAdd(ghist + sl, 1ull);
            }
        }
      }
    }
  }
  uint32_t bits;
  double E;
  int emax;
  int cf[SZ];
  uint32_t u[SZ];
  zfp_block<D, false>(blk, minexp, bits, E, emax, cf, u);
  tbits = act ? bits : 0u;
  terr = act ? E : 0.0;
}

// Move the CTA's smem histogram (lane copies + packed table) into the global histogram
// and clear it.  Called by the consumer threads (tid < nthr) after a consumer barrier.
template <int D>
__device__ __forceinline__ void tile_hist_flush(unsigned int *hist, unsigned int *tbl,
                                                const int *tbl_used, int tbl_mark,
                                                unsigned long long *ghist,
                                                int tid, int nthr) {
  using Cfg = TileCfg<D>;
  for (int i = tid; i < kHBins; i += nthr) {
    unsigned long long c = 0;
#pragma unroll
    for (int k = 0; k < Cfg::COPIES; ++k) {
      c += hist[k * kHStride + i];
      hist[k * kHStride + i] = 0u;
    }
    if (c) atomicAdd(ghist + (kCenter - kHBins / 2) + i, c);
  }
  // the flag holds the mark of the last flush interval that used the table (a mark per
  // interval, so nobody has to reset it between a flush and the next codes)
  if (*tbl_used != tbl_mark) return;    // no code outside the lane-copy window: table is zero
  for (int i = tid; i < Cfg::TB; i += nthr) {
    const uint32_t v = tbl[i];
    if (v) {
      tbl[i] = 0u;
      atomicAdd(ghist + (kCenter - Cfg::TB / 2) + i, (unsigned long long)v);
    }
  }
}

// TMA descriptor of a field for the tile box (sel_tile.cu)
int make_tile_map(CUtensorMap *map, const float *x, const Geo &g);

}  // namespace sel
