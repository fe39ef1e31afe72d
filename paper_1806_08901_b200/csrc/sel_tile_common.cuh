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
#define SEL_CW2 16             // (+ producer, release and 2 range warps in k_batch: 20 warps at 96 registers)
#endif
#ifndef SEL_STAGES2
#define SEL_STAGES2 2
#endif
#ifndef SEL_W2
#define SEL_W2 8192            // shared-memory histogram window (bins), 2D
#endif
#ifndef SEL_W3
#define SEL_W3 12288           // 3D
#endif
#ifndef SEL_BR2
#define SEL_BR2 2              // 2D: block rows per consumer warp and tile task
#endif
#ifndef SEL_CW3
#define SEL_CW3 8
#endif
#ifndef SEL_STAGES3
#define SEL_STAGES3 2
#endif

constexpr int kBoxK = 4 * 32 + 4;             // 132 floats: 4 halo columns (last one used) + 128
constexpr int kChunk = 1024;                  // window flush granule (bins)

template <int D>
struct TileCfg {
  static constexpr int CW = D == 3 ? SEL_CW3 : SEL_CW2;           // consumer warps
  static constexpr int THREADS = (CW + 1) * 32;
  static constexpr int BR = D == 2 ? SEL_BR2 : 1;                 // block rows per warp
  static constexpr int ROWS = CW * BR;                            // block rows per tile
  static constexpr int BOXJ = 4 * ROWS + 1;                       // halo row + 4 per block row
  static constexpr int BOXI = D == 3 ? 5 : 1;                     // halo plane + 4 (3D)
  static constexpr int PLANE = kBoxK * BOXJ;                      // floats per smem plane
  static constexpr uint32_t STAGE_BYTES = PLANE * BOXI * 4;
  static constexpr int STAGE_FLOATS = ((STAGE_BYTES + 127) & ~127) / 4;
  static constexpr int STAGES = D == 3 ? SEL_STAGES3 : SEL_STAGES2;
  // One CTA-wide histogram window of W u32 bins in shared memory, codes [-W/2, W/2),
  // one copy: smem atomic increments with unused results compile to ATOMS.POPC.INC,
  // which merges the lanes of a warp that hit the same bin (measured: 1 copy is as fast
  // as 2 or 8 lane-replicated copies on the smooth configs).  Word W is the pad bin that
  // out-of-window codes (counted by the far path) and inactive lanes increment.
  static constexpr int W = D == 3 ? SEL_W3 : SEL_W2;
  static constexpr int HIST_WORDS = W + 4;
  static constexpr uint32_t kWOff = kSlotOff + (uint32_t)(kCenter - W / 2);   // bits(q+M) -> bin
  static constexpr size_t SMEM = 128 + (size_t)STAGES * STAGE_FLOATS * 4 + HIST_WORDS * 4 +
                                 STAGES * 48 + 16;
  static_assert(W % kChunk == 0 && (kCenter - W / 2 + 1) % 4 == 0, "window alignment");
  static_assert(SMEM <= 232448, "shared memory");
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
  // the left neighbour straight from the tile (a 16-byte lane stride: 4 wavefronts, but one
  // instruction instead of a broadcast load + shuffle + select; the LSU has the headroom)
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const float4 q = *reinterpret_cast<const float4 *>(prow + r * kBoxK + 4 + 4 * lane);
    v[r][0] = q.x; v[r][1] = q.y; v[r][2] = q.z; v[r][3] = q.w;
    h[r] = prow[r * kBoxK + 3 + 4 * lane];
  }
}

// SZ code of one residual: b = bits(q + M) (reading R5, see sel_device.cuh), w = its
// bin in the window; one unconditional increment (no divergence): out-of-window values
// (and every value of a lane whose r_f is NaN, i.e. an inactive lane) land in the pad bin
// W, ignored at the flush.
template <int D>
__device__ __forceinline__ uint32_t sz_win(float d, float r_f, unsigned int *win) {
  const uint32_t b = __float_as_uint(__fadd_rn(__fmul_rn(d, r_f), kMagic));
  const uint32_t w = b - TileCfg<D>::kWOff;
  atomicAdd(win + min(w, (uint32_t)TileCfg<D>::W), 1u);
  return w;
}

// Codes of one row of 4 that fell outside the window (wide distributions: noise, fronts):
// one warp-uniform branch per row; each goes to the global histogram, or to the overflow
// count (slot 65,535, R5).  act: the lane's values are real SZ points.
template <int D, typename GH>
__device__ __forceinline__ void sz_far(const uint32_t (&w)[4], uint32_t any, bool act, GH *ghist,
                                       unsigned int &ovf) {
  using Cfg = TileCfg<D>;
  if (__any_sync(0xffffffffu, act && any >= (uint32_t)Cfg::W)) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (act && w[c] >= (uint32_t)Cfg::W) {
        const uint32_t sl = w[c] + (Cfg::kWOff - kSlotOff);
        if (sl > 65534u) ++ovf;
        else atomicAdd(ghist + sl, (GH)1);
      }
  }
}

__device__ __forceinline__ float lane_rf(bool act, float r_f) {   // NaN: every code -> pad bin
  return act ? r_f : __uint_as_float(0x7fc00000u);
}


// Consumer work of one tile task (block-layer bi, tile row btj, tile column btk; warp-level:
// every consumer warp of the CTA calls it for the same tile).  S: the tile's smem stage.  Adds the SZ codes to the CTA's histogram
// (lane copies / packed table / ghist / ovf) and returns the lane's block bits/error.
// ROLE: 0 = SZ then ZFP by the same warp; 1 = the SZ half only, 2 = the ZFP half only (the
// two halves read the tile independently, so they can run on different warps).
template <int D, bool DBG, typename GH = unsigned long long, int ROLE = 0>
__device__ __forceinline__ void tile_consume(const float *S, int btk, int btj, int bi,
                                             const TileGeo &tg, int warp,
                                             int lane, bool ok, float r_f, int minexp,
                                             unsigned int *win,
                                             GH *ghist,
                                             unsigned int &ovf, const DebugPtrs &dbg,
                                             uint64_t &tbits, double &terr) {
  using Cfg = TileCfg<D>;
  constexpr int SZ = Tab<D>::SIZE;
  constexpr int NPL = D == 3 ? 4 : 1;
  // per-axis extents and block coordinates fit 32 bits (tile_supported); only the debug
  // dumps form 64-bit linear indices
  const int n0 = (int)tg.n[0], n1 = (int)tg.n[1], n2 = (int)tg.n[2];
  const int bk = btk * 32 + lane;
  tbits = 0;
  terr = 0.0;
#pragma unroll 1
  for (int rb = 0; rb < Cfg::BR; ++rb) {          // the warp's block rows, in order
    const int wr = warp * Cfg::BR + rb;           // block row within the tile
    const int bj = btj * Cfg::ROWS + wr;
    if (ok && bj < tg.nb[1]) {
      const bool activeK = bk < tg.nb[2];
      const int I0 = 4 * bi, J0 = 4 * bj, K0 = 4 * bk;
      const float *wrow = S + (4 * wr) * kBoxK;     // smem row of j = J0 - 1 (plane 0)
      const float rf = lane_rf(activeK, r_f);
      // ---------------- SZ: nested differences on the tile (R4), codes -> histogram (R5)
      static_assert(D == 3 || ROLE == 0, "split roles: 3D only");
      float blk2[D == 2 ? 16 : 1];   // 2D: the ZFP block is rows 1..4 of the SZ plane
      if constexpr (ROLE != 2) {
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
      // Blocks away from the far edges and the field origin (warp-uniform) skip the per-row
      // bound / origin checks and the edge replication.
      const bool edge = J0 + 4 > n1 || (D == 3 && I0 + 4 > n0) || (btk == 0 && J0 == 0 && I0 == 0);
      auto rows = [&](auto EDGE, int i, const float (&v)[5][4], const float (&h)[5], float (&d1up)[4]) {
        constexpr bool E = decltype(EDGE)::value;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int j = J0 + r;
          if (E && (i >= n0 || j >= n1)) break;       // padded rows/planes: no SZ point
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
            w[c] = sz_win<D>(d, rf, win);
            any |= w[c];
          }
          // the field origin is stored verbatim, not coded (R4): undo its count
          const bool orow = E && (i == 0) && (j == 0) && (btk == 0);
          if (orow && lane == 0) {
            if (w[0] < (uint32_t)Cfg::W) atomicSub(win + w[0], 1u);
            w[0] = 0u;
          }
          if constexpr (DBG) {
            if (activeK) {
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                if (orow && lane == 0 && c == 0) continue;
                const uint32_t sl = w[c] + (Cfg::kWOff - kSlotOff);
                dbg.codes[((int64_t)i * n1 + j) * n2 + K0 + c] = sl > 65534u ? kOvfSlot : (int32_t)sl;
              }
            }
          }
          sz_far<D>(w, any, activeK, ghist, ovf);
        }
      };
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
              blk2[4 * r + c] = (r == 0 || !edge || J0 + r < n1) ? v[r + 1][c] : blk2[4 * (r - 1) + c];
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) d1up[c] = v[0][c] - (c ? v[0][c - 1] : h[0]);
        if (edge) rows(std::true_type{}, i, v, h, d1up);
        else rows(std::false_type{}, i, v, h, d1up);
      }
      }
      // ---------------- ZFP on the lane's block, edge-replicated at the far edges (R17)
      if (ROLE != 1 && activeK) {
        float blk[SZ];
        if constexpr (D == 2) {
#pragma unroll
          for (int n = 0; n < 16; ++n) blk[n] = blk2[n];
        } else {
          const float *bbase = S + Cfg::PLANE + (4 * wr + 1) * kBoxK + 4 + 4 * lane;
          if (J0 + 4 <= n1 && I0 + 4 <= n0) {        // interior (warp-uniform): fixed offsets
#pragma unroll
            for (int p = 0; p < NPL; ++p)
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                const float4 q = *reinterpret_cast<const float4 *>(bbase + p * Cfg::PLANE + r * kBoxK);
                const int o = (p * 4 + r) * 4;
                blk[o] = q.x; blk[o + 1] = q.y; blk[o + 2] = q.z; blk[o + 3] = q.w;
              }
          } else {
#pragma unroll
            for (int p = 0; p < NPL; ++p) {
              const int ic = min(I0 + p, n0 - 1) - I0;          // 0..3, edge-replicated
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                const int jc = min(J0 + r, n1 - 1) - J0;         // 0..3
                const float4 q = *reinterpret_cast<const float4 *>(bbase + ic * Cfg::PLANE + jc * kBoxK);
                const int o = (p * 4 + r) * 4;
                blk[o] = q.x; blk[o + 1] = q.y; blk[o + 2] = q.z; blk[o + 3] = q.w;
              }
            }
          }
        }
        uint32_t bits;
        double E;
        int emax;
        int cf[SZ];
        uint32_t u[SZ];
        zfp_block<D, DBG>(blk, minexp, bits, E, emax, cf, u);
        tbits += bits;
        terr += E;
        if constexpr (DBG) {
          const int64_t tb = (D == 3 ? ((int64_t)bi * tg.nb[1] + bj) : (int64_t)bj) * tg.nb[2] + bk;   // block index
          dbg.emax[tb] = emax; dbg.bits[tb] = bits; dbg.err[tb] = E;
#pragma unroll
          for (int n = 0; n < SZ; ++n) { dbg.coef[tb * SZ + n] = cf[n]; dbg.uword[tb * SZ + n] = u[n]; }
        }
      }
    }
  }
}

// Sampled-block task (strides > 1; k_batch): lane = processed block t (act: t < n_pb),
// read with its halo from global memory (L2: the range pass just streamed the field),
// codes into the same smem histogram as a tile task, ZFP block in registers.  Every lane
// of the warp runs (inactive lanes on a clamped block, contributing nothing) so the
// warp-uniform out-of-window branch stays uniform.
template <int D, typename GH>
__device__ __forceinline__ void sampled_consume(const float *__restrict__ x, const Geo &g,
                                                int64_t t, bool act, float r_f, int minexp,
                                                unsigned int *win,
                                                GH *ghist, unsigned int &ovf,
                                                uint64_t &tbits, double &terr) {
  using Cfg = TileCfg<D>;
  constexpr int SZ = Tab<D>::SIZE;
  constexpr int PL = D == 3 ? 4 : 1;
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
        w[c] = sz_win<D>(d, valid ? r_f : __uint_as_float(0x7fc00000u), win);
        w[c] = valid ? w[c] : 0u;
        any |= w[c];
      }
      sz_far<D>(w, any, true, ghist, ovf);
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

// Move the CTA's smem window into the global (u64) histogram and clear it (k_tile, at
// the end of its field).  Called by the consumer threads (tid < nthr) after a barrier.
template <int D>
__device__ __forceinline__ void tile_hist_flush(unsigned int *win, unsigned long long *ghist, int tid,
                                                int nthr) {
  using Cfg = TileCfg<D>;
  for (int i = tid; i < Cfg::W; i += nthr) {
    const unsigned int c = win[i];
    if (c) {
      win[i] = 0u;
      atomicAdd(ghist + (kCenter - Cfg::W / 2) + i, (unsigned long long)c);
    }
  }
}

// TMA descriptor of a field for the tile box (sel_tile.cu)
int make_tile_map(CUtensorMap *map, const float *x, const Geo &g);

}  // namespace sel
