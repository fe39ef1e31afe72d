// sel_tile3q.cuh -- the 3D tile consumer with four lanes per 4x4x4 block.
//
// One lane per 3D block needs 64 values in registers (~160 registers) and 8 KB of stage
// per warp, which held the 3D kernels to 8 consumer warps per SM.  Here lane (b, q) =
// (lane >> 2, lane & 3) owns plane z = q of block b (16 values, like a 2D lane), a warp
// covers 8 blocks along k, and a tile is 4 warps along k x CW/4 warps along j (one block
// layer): 16 consumer warps fit.  Per block:
//   SZ (R4/R5): the lane forms the nested differences of its plane from smem planes q+1
//     (its own) and q (the one below; plane 0 of the stage is the halo), rows/columns
//     with their halo row/column -- no state carried across planes.
//   ZFP (R8-R14): exponent by a 4-lane max; BFP; x- and y-lifts in registers; the z-lift
//     after a 4x4 transpose through a per-warp scratch (lane q then holds y = q, all x,
//     z); negabinary; the truncation error per lane (weight g(y=q) x class of (x, z));
//     the group-testing count (R13) after a second scatter into sequency order, so that
//     lane q holds sequency positions 16q..16q+15: a local suffix-max chain seeded with
//     the maximum of the lanes above, combined with three 4-lane reductions.
// Every per-block quantity is the same integer / the same sum as the one-lane routine
// (the debug dumps are compared block by block with the oracle).
#pragma once

namespace sel {

// scratch per warp: 8 blocks x 4 planes x (16 + 4 pad) words (conflict-free 128-bit rows)
constexpr int kScrBlock = 80;
constexpr int kScrWarp = 8 * kScrBlock;

struct Perm3 {                       // sequency position of natural 3D index n = x + 4y + 16z
  int pos[64];
};
__host__ __device__ constexpr Perm3 make_pos3() {
  Perm3 p{};
  constexpr auto perm = Tab<3>::make_perm();
  for (int j = 0; j < 64; ++j) p.pos[perm.v[j]] = j;
  return p;
}
// scratch word of sequency position j (the same padding as the transpose layout)
__device__ __forceinline__ constexpr int scr_seq(int j) { return j + (j >> 4) * 4; }

template <bool DBG, int TBS>
__device__ __forceinline__ void tile_consume_3q(const float *S, int btk, int btj, int bi,
                                                const TileGeo &tg, int warp, int lane, bool ok,
                                                float r_f, int minexp, unsigned int *hlane,
                                                unsigned int *htrash, unsigned int *tbl,
                                                int *tbl_used, int tbl_mark,
                                                unsigned long long *ghist, unsigned int &ovf,
                                                const DebugPtrs &dbg, unsigned int *scr,
                                                uint64_t &tbits, double &terr) {
  using Cfg = TileCfg<3>;
  constexpr int WJ = Cfg::WJ;
  constexpr int PLANE = Cfg::PLANE;
  const int n0 = (int)tg.n[0], n1 = (int)tg.n[1], n2 = (int)tg.n[2];
  const int wk = warp & 3, wj = warp >> 2;
  const int b = lane >> 2, q = lane & 3;
  const int bj = btj * WJ + wj;
  const int bk = btk * 32 + wk * 8 + b;
  tbits = 0;
  terr = 0.0;
  if (!ok || bj >= tg.nb[1]) return;                 // warp-uniform
  const bool activeK = bk < tg.nb[2];
  const int I0 = 4 * bi, J0 = 4 * bj, K0 = 4 * bk;
  const int i = I0 + q;                              // this lane's plane
  unsigned int *const hcopy = activeK ? hlane : htrash;
  // ---------------- SZ (R4, R5)
  const int col = 4 + 32 * wk + 4 * b;               // smem column of k = K0
  float v[5][4];                                     // plane q+1 (own), rows j = J0-1 .. J0+3
  float D2p[4][4];                                   // nested row differences of plane q
  {
    const float *pl = S + q * PLANE + (4 * wj) * kBoxK;      // plane i - 1
    float u[5][4], hu[5];
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const float4 t = *reinterpret_cast<const float4 *>(pl + r * kBoxK + col);
      u[r][0] = t.x; u[r][1] = t.y; u[r][2] = t.z; u[r][3] = t.w;
      hu[r] = pl[r * kBoxK + col - 1];
    }
    float d1p[5][4];
#pragma unroll
    for (int r = 0; r < 5; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) d1p[r][c] = u[r][c] - (c ? u[r][c - 1] : hu[r]);
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) D2p[r][c] = d1p[r + 1][c] - d1p[r][c];
  }
  {
    const float *pl = S + (q + 1) * PLANE + (4 * wj) * kBoxK;   // plane i
    float hv[5];
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const float4 t = *reinterpret_cast<const float4 *>(pl + r * kBoxK + col);
      v[r][0] = t.x; v[r][1] = t.y; v[r][2] = t.z; v[r][3] = t.w;
      hv[r] = pl[r * kBoxK + col - 1];
    }
    float d1up[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) d1up[c] = v[0][c] - (c ? v[0][c - 1] : hv[0]);
    const bool orig = (I0 == 0) && (J0 == 0) && (K0 == 0) && q == 0;   // block of the origin
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int j = J0 + r;
      const bool rowok = i < n0 && j < n1;           // padded rows / planes: no SZ point
      uint32_t w[4];
      uint32_t any = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float d1 = v[r + 1][c] - (c ? v[r + 1][c - 1] : hv[r + 1]);
        const float d2 = d1 - d1up[c];
        d1up[c] = d1;
        const float d = d2 - D2p[r][c];
        // no code for padded points and the origin (stored verbatim, R4): their count goes
        // to the trash copy, w = 0 keeps them out of the out-of-window path
        const bool valid = rowok && !(orig && r == 0 && c == 0);
        w[c] = sz_win(d, r_f, valid ? hcopy : htrash);
        w[c] = valid ? w[c] : 0u;
        any |= w[c];
      }
      if constexpr (DBG) {
        if (activeK && rowok) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (orig && r == 0 && c == 0) continue;
            const uint32_t sl = w[c] + (kHOff - kSlotOff);
            dbg.codes[((int64_t)i * n1 + j) * n2 + K0 + c] = sl > 65534u ? kOvfSlot : (int32_t)sl;
          }
        }
      }
      // out-of-window codes: one warp-uniform branch per row (see tile_consume)
      if (__any_sync(0xffffffffu, activeK && rowok && any >= (uint32_t)kHBins)) {
        uint32_t far = 0u;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          constexpr uint32_t kTOffS = kSlotOff + (uint32_t)(kCenter - TBS / 2);
          const uint32_t tb = w[c] + (kHOff - kTOffS);
          const bool out = activeK && rowok && w[c] >= (uint32_t)kHBins;
          if (out && tb < (uint32_t)TBS) atomicAdd(tbl + tb, 1u);
          far |= (out && tb >= (uint32_t)TBS) ? (1u << c) : 0u;
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
  // ---------------- ZFP on block b: this lane's plane, edge-replicated (R17)
  float x[16];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) x[4 * r + c] = (r == 0 || J0 + r < n1) ? v[r + 1][c] : x[4 * (r - 1) + c];
  if (I0 + 3 >= n0) {                                // last block layer: planes past n0 copy n0-1
    const int qlast = n0 - 1 - I0;                   // uniform over the warp
#pragma unroll
    for (int n = 0; n < 16; ++n) {
      const float t = __shfl_sync(0xffffffffu, x[n], (lane & ~3) | qlast);
      if (q > qlast) x[n] = t;
    }
  }
  float m = 0.0f;
#pragma unroll
  for (int n = 0; n < 16; ++n) m = fmaxf(m, fabsf(x[n]));
  m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
  m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
  // lanes of inactive blocks (past nb[2]) run along on their (zero-filled) data but
  // contribute nothing; every lane takes part in the shuffles / scratch exchanges
  int bits_part = 0;                                 // this lane's share of the block's bits
                                                     // (may be negative; the 4 lanes sum to it)
  double E = 0.0;
  int emax = -127;
  int cf[16];
  uint32_t us[16];                                   // sequency positions 16q .. 16q+15
#pragma unroll
  for (int n = 0; n < 16; ++n) { cf[n] = 0; us[n] = 0u; }
  const bool nz = m != 0.0f;                         // uniform over the block
  if (nz) emax = (int)(__float_as_uint(m) >> 23) - 126;
  // block floating point (R9), two-step scale below 2^-97
  if (emax >= -97) {
    const float sc = __uint_as_float((uint32_t)(157 - emax) << 23);
#pragma unroll
    for (int n = 0; n < 16; ++n) cf[n] = __float2int_rz(__fmul_rn(x[n], sc));
  } else if (nz) {
    const float sc = __uint_as_float((uint32_t)(93 - emax) << 23);
#pragma unroll
    for (int n = 0; n < 16; ++n) cf[n] = __float2int_rz(__fmul_rn(__fmul_rn(x[n], 0x1p64f), sc));
  }
  // x- then y-lifts on the plane (R8)
#pragma unroll
  for (int r = 0; r < 4; ++r) fwd_lift(cf[4 * r], cf[4 * r + 1], cf[4 * r + 2], cf[4 * r + 3]);
#pragma unroll
  for (int c = 0; c < 4; ++c) fwd_lift(cf[c], cf[4 + c], cf[8 + c], cf[12 + c]);
  // transpose: lane (b, q) writes plane z = q as rows y, reads row y = q of every plane z
  unsigned int *const sb = scr + b * kScrBlock;
#pragma unroll
  for (int r = 0; r < 4; ++r)
    *reinterpret_cast<int4 *>(sb + q * 20 + r * 4) = make_int4(cf[4 * r], cf[4 * r + 1], cf[4 * r + 2], cf[4 * r + 3]);
  __syncwarp();
  int t[4][4];                                       // t[z][x] at y = q
#pragma unroll
  for (int z = 0; z < 4; ++z) {
    const int4 rr = *reinterpret_cast<const int4 *>(sb + z * 20 + q * 4);
    t[z][0] = rr.x; t[z][1] = rr.y; t[z][2] = rr.z; t[z][3] = rr.w;
  }
  __syncwarp();
  // z-lift (R8)
#pragma unroll
  for (int c = 0; c < 4; ++c) fwd_lift(t[0][c], t[1][c], t[2][c], t[3][c]);
  // negabinary (R11); natural index n = x + 4 q + 16 z
  uint32_t u[4][4];
#pragma unroll
  for (int z = 0; z < 4; ++z)
#pragma unroll
    for (int c = 0; c < 4; ++c) u[z][c] = to_negabinary(t[z][c]);
  int prec = emax - minexp + 2 * (3 + 1);
  prec = prec < 0 ? 0 : (prec > 32 ? 32 : prec);
  const int kmin = 32 - prec;
  // gain-weighted truncation error of this lane's 16 coefficients (R14): weight =
  // g(x) g(y) g(z), g = (4, 5, 4, 13/4); y = q fixed per lane, (x, z) classes as in 2D
  if (nz) {
    const double gq = q == 1 ? 5.0 : (q == 3 ? 3.25 : 4.0);
    if (kmin >= 30) {
      const uint32_t low = kmin >= 32 ? 0xffffffffu : ((1u << kmin) - 1u);
      const uint32_t Mk = 0xAAAAAAAAu & low;
      double s = 0.0;
#pragma unroll
      for (int z = 0; z < 4; ++z)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double w2 = Tab<2>::gain(c + 4 * z);
          const long long e = (long long)((u[z][c] & low) ^ Mk) - (long long)Mk;
          const double ed = (double)e;
          s = __dadd_rn(s, __dmul_rn(w2, __dmul_rn(ed, ed)));
        }
      E = __dmul_rn(__dmul_rn(s, gq), pow2d(2 * (emax - 30)));
    } else {
      const uint32_t low = (1u << kmin) - 1u;
      const uint32_t Mk = 0xAAAAAAAAu & low;
      unsigned long long acc[Tab<2>::NCLS];
#pragma unroll
      for (int k = 0; k < Tab<2>::NCLS; ++k) acc[k] = 0ull;
      static_for<0, 16>([&](auto N) {
        constexpr int n2d = decltype(N)::value;      // x + 4 z
        constexpr int cl = Tab<2>::cls_of(n2d);
        const int e = (int)((u[n2d >> 2][n2d & 3] & low) ^ Mk) - (int)Mk;
        acc[cl] += (unsigned long long)((long long)e * (long long)e);
      });
      double s = 0.0;
      static_for<0, Tab<2>::NCLS>([&](auto C) {
        constexpr int cl = decltype(C)::value;
        s = __dadd_rn(s, __dmul_rn(Tab<2>::cls_weight(cl), (double)acc[cl]));
      });
      E = __dmul_rn(__dmul_rn(s, gq), pow2d(2 * (emax - 30)));
    }
  }
  // sequency order (R10): scatter the 16 words to their positions, read back 16q..16q+15
  {
    const int sh = 8 * q;
    static_for<0, 16>([&](auto N) {
      constexpr int n2d = decltype(N)::value;        // x + 4 z
      constexpr int c = n2d & 3, z = n2d >> 2;
      constexpr Perm3 P = make_pos3();
      // sequency positions of (x = c, y = 0..3, z) packed in bytes; pick y = q
      constexpr uint32_t pk = (uint32_t)P.pos[c + 16 * z] | ((uint32_t)P.pos[c + 4 + 16 * z] << 8) |
                              ((uint32_t)P.pos[c + 8 + 16 * z] << 16) |
                              ((uint32_t)P.pos[c + 12 + 16 * z] << 24);
      const int j = (int)((pk >> sh) & 0xffu);
      sb[scr_seq(j)] = u[z][c];
    });
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 rr = *reinterpret_cast<const uint4 *>(sb + q * 20 + 4 * k);
      us[4 * k] = rr.x; us[4 * k + 1] = rr.y; us[4 * k + 2] = rr.z; us[4 * k + 3] = rr.w;
    }
    __syncwarp();
  }
  // group-testing count (R13), the closed form of sel_device.cuh split over the 4 lanes:
  // lane q runs the chain over positions 16q..16q+15 seeded with R = max(kmin, max f above)
  {
    int fmaxl = -1;
#pragma unroll
    for (int n = 0; n < 16; ++n) fmaxl = max(fmaxl, flo(us[n]));
    const int a1 = __shfl_down_sync(0xffffffffu, fmaxl, 1);
    const int a2 = __shfl_down_sync(0xffffffffu, fmaxl, 2);
    const int a3 = __shfl_down_sync(0xffffffffu, fmaxl, 3);
    int above = -1;
    if (q < 3) above = max(above, a1);
    if (q < 2) above = max(above, a2);
    if (q < 1) above = max(above, a3);
    int R = max(kmin, above), sR = 0;
    uint32_t cm = 0u;
#pragma unroll
    for (int n = 15; n >= 0; --n) {
      const int f = flo(us[n]);
      if (f >= R) cm |= 1u << n;
      R = max(R, f);
      sR += R;
    }
    // block terms: last position of C (z = 63 - last), f_L of position 63 (lane 3)
    int last = cm ? 16 * q + flo(cm) : -1;
    last = max(last, __shfl_xor_sync(0xffffffffu, last, 1));
    last = max(last, __shfl_xor_sync(0xffffffffu, last, 2));
    if (nz && prec > 0) {
      bits_part = sR + __popc(cm);
      if (q == 3) {
        const int fL = flo(us[15]);
        const int t3 = 32 - max(fL + 1, kmin) - (fL >= kmin ? 1 : 0);
        bits_part += 9 - 64 * (kmin - 1) + t3 - (63 - last);
      }
    } else {
      bits_part = q == 3 ? 1 : 0;                    // empty block or p == 0: one bit
    }
  }
  if (activeK) {
    tbits = (uint64_t)(int64_t)bits_part;          // the u64 task sum wraps back exactly
    terr = E;
  }
  if constexpr (DBG) {
    uint32_t bsum = (uint32_t)bits_part;
    bsum += __shfl_xor_sync(0xffffffffu, bsum, 1);
    bsum += __shfl_xor_sync(0xffffffffu, bsum, 2);
    double es = E;                                   // block error: the lanes' sum
    es = __dadd_rn(es, __shfl_xor_sync(0xffffffffu, es, 1));
    es = __dadd_rn(es, __shfl_xor_sync(0xffffffffu, es, 2));
    if (activeK) {
      const int64_t tb = ((int64_t)bi * tg.nb[1] + bj) * tg.nb[2] + bk;
      if (q == 0) { dbg.emax[tb] = emax; dbg.bits[tb] = bsum; dbg.err[tb] = es; }
#pragma unroll
      for (int z = 0; z < 4; ++z)
#pragma unroll
        for (int c = 0; c < 4; ++c) dbg.coef[tb * 64 + c + 4 * q + 16 * z] = nz ? t[z][c] : 0;
#pragma unroll
      for (int n = 0; n < 16; ++n) dbg.uword[tb * 64 + 16 * q + n] = nz ? us[n] : 0u;
    }
  }
}

}  // namespace sel
