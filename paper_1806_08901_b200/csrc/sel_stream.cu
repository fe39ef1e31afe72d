// sel_stream.cu -- SURVEY 8(f) N3, the ZFP branch of Alg. 1 lines 11-15:
// "perform ZFP compression on X_i with absolute error bound eb" -- the fixed-accuracy
// stream whose per-block lengths the estimator already counts exactly (R13).
//
// Layout (the oracle's orc_zfp_stream, bit for bit): per processed block in row-major
// order, 1 bit 0 if the block is empty or p = 0; else 1 bit 1, 8 bits emax + 127, then the
// group-testing embedded code of bit planes 31..kmin (R13's coder: per plane the bits of
// the n already-significant coefficients verbatim, then group tests); bits packed LSB
// first (bit i of the stream = bit i % 32 of 32-bit word i / 32, little endian).
//
// Launches: k_minmax -> k_zbits (per-block lengths) -> k_scan_sum -> k_scan_top (CTA
// bases, total) -> [host reads the total] -> k_zwrite (every block writes its bits at its
// offset; a block's first and last words are shared with its neighbours: atomicOr).
#include "sel_device.cuh"

namespace sel {

constexpr int kScanB = 1024;       // blocks per scan / writer CTA (256 threads x 4)

// per processed block t: the exact stream length of the block (header + EC bits)
template <int D, bool VEC>
__global__ void __launch_bounds__(256) k_zbits(const float *__restrict__ x, Geo g, const Params *prm_,
                                               uint32_t *bits) {
  constexpr int SZ = Tab<D>::SIZE;
  constexpr int PL = D == 3 ? 4 : 1;
  constexpr int RW = D >= 2 ? 4 : 1;
  const Params prm = *prm_;
  if (prm.status != SEL_OK) return;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < g.n_pb; t += gstride) {
    const int64_t p2 = t % g.npb[2];
    const int64_t q = t / g.npb[2];
    const int64_t p1 = q % g.npb[1];
    const int64_t p0 = q / g.npb[1];
    float blk[SZ];
#pragma unroll
    for (int p = 0; p < PL; ++p)
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        float v[4], h;
        load_row<VEC>(x, g, 4 * p0 * g.s[0] + p, 4 * p1 * g.s[1] + r, 4 * p2 * g.s[2], v, h);
#pragma unroll
        for (int c = 0; c < 4; ++c) blk[(p * RW + r) * 4 + c] = v[c];
      }
    uint32_t b;
    double E;
    int emax;
    int cf[SZ];
    uint32_t u[SZ];
    zfp_block<D, false>(blk, prm.minexp, b, E, emax, cf, u);
    bits[t] = b;
  }
}

// CTA c: sum of the lengths of blocks [c kScanB, (c + 1) kScanB)
__global__ void __launch_bounds__(256) k_scan_sum(const uint32_t *bits, int64_t n, unsigned long long *csum) {
  const int64_t b0 = (int64_t)blockIdx.x * kScanB;
  unsigned long long s = 0;
  for (int k = threadIdx.x; k < kScanB; k += blockDim.x)
    if (b0 + k < n) s += bits[b0 + k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  __shared__ unsigned long long sw[8];
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) s += sw[w];
    csum[blockIdx.x] = s;
  }
}

// one CTA: exclusive scan of the CTA sums (in place) and the stream total
__global__ void __launch_bounds__(1024) k_scan_top(unsigned long long *csum, int nc, unsigned long long *total) {
  __shared__ unsigned long long carry;
  __shared__ unsigned long long sw[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nc; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const unsigned long long v = i < nc ? csum[i] : 0ull;
    // inclusive warp scan, then across warps
    unsigned long long x = v;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) sw[wid] = x;
    __syncthreads();
    if (wid == 0) {
      unsigned long long w = lane < (int)(blockDim.x >> 5) ? sw[lane] : 0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      sw[lane] = w;   // inclusive prefix of the warp sums
    }
    __syncthreads();
    const unsigned long long excl = carry + (wid ? sw[wid - 1] : 0ull) + x - v;
    if (i < nc) csum[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// bit writer into 32-bit words (LSB first) of a zeroed buffer; a block's first word (when
// the block does not start on a word boundary) and its last, partial word may be shared
// with its neighbours: atomicOr; every word in between is the block's own: a plain store
struct BitWriter {
  uint32_t *out;
  unsigned long long word;
  int off;                      // bits of cur already filled (0..31)
  unsigned long long cur;
  bool shared_word;             // the word being filled started before this block
  __device__ __forceinline__ void init(uint32_t *o, unsigned long long pos) {
    out = o;
    word = pos >> 5;
    off = (int)(pos & 31);
    cur = 0ull;
    shared_word = off != 0;
  }
  __device__ __forceinline__ void put(uint32_t v, int n) {   // n <= 32 bits of v
    if (n <= 0) return;
    const unsigned long long m = n == 32 ? 0xffffffffull : ((1ull << n) - 1ull);
    cur |= ((unsigned long long)v & m) << off;
    off += n;
    if (off >= 32) {
      if (shared_word) atomicOr(out + word, (uint32_t)cur);
      else out[word] = (uint32_t)cur;
      shared_word = false;
      cur >>= 32;
      off -= 32;
      ++word;
    }
  }
  __device__ __forceinline__ void put64(unsigned long long v, int n) {   // n <= 64
    if (n > 32) {
      put((uint32_t)v, 32);
      put((uint32_t)(v >> 32), n - 32);
    } else {
      put((uint32_t)v, n);
    }
  }
  __device__ __forceinline__ void zeros(int n) {
    while (n > 32) { put(0u, 32); n -= 32; }
    put(0u, n);
  }
  __device__ __forceinline__ void flush() {
    if (off > 0) atomicOr(out + word, (uint32_t)cur);
  }
};

// writer CTA c: blocks [c kScanB, +kScanB), 4 consecutive per thread; offsets = the CTA
// base + an in-CTA exclusive scan of the lengths
template <int D, bool VEC>
__global__ void __launch_bounds__(256) k_zwrite(const float *__restrict__ x, Geo g, const Params *prm_,
                                                const uint32_t *bits, const unsigned long long *cbase,
                                                uint32_t *out) {
  constexpr int SZ = Tab<D>::SIZE;
  constexpr int PL = D == 3 ? 4 : 1;
  constexpr int RW = D >= 2 ? 4 : 1;
  const Params prm = *prm_;
  if (prm.status != SEL_OK) return;
  const int64_t b0 = (int64_t)blockIdx.x * kScanB + 4 * threadIdx.x;
  unsigned long long mine = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (b0 + k < g.n_pb) mine += bits[b0 + k];
  // exclusive scan of `mine` over the CTA
  unsigned long long x_ = mine;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x_, o);
    if (lane >= o) x_ += y;
  }
  __shared__ unsigned long long sw[8];
  if (lane == 31) sw[wid] = x_;
  __syncthreads();
  unsigned long long pre = 0;
  for (int w = 0; w < wid; ++w) pre += sw[w];
  unsigned long long pos = cbase[blockIdx.x] + pre + x_ - mine;
  for (int k = 0; k < 4; ++k) {
    const int64_t t = b0 + k;
    if (t >= g.n_pb) break;
    const int64_t p2 = t % g.npb[2];
    const int64_t q = t / g.npb[2];
    const int64_t p1 = q % g.npb[1];
    const int64_t p0 = q / g.npb[1];
    float blk[SZ];
#pragma unroll
    for (int p = 0; p < PL; ++p)
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        float v[4], h;
        load_row<VEC>(x, g, 4 * p0 * g.s[0] + p, 4 * p1 * g.s[1] + r, 4 * p2 * g.s[2], v, h);
#pragma unroll
        for (int c = 0; c < 4; ++c) blk[(p * RW + r) * 4 + c] = v[c];
      }
    BitWriter bw;
    bw.init(out, pos);
    int emax;
    int cf[SZ];
    int prec = 0;
    if (zfp_transform<D>(blk, emax, cf)) {
      prec = emax - prm.minexp + 2 * (D + 1);
      prec = prec < 0 ? 0 : (prec > 32 ? 32 : prec);
    }
    if (prec == 0) {
      bw.put(0u, 1);                           // empty block or nothing kept
    } else {
      bw.put(1u, 1);
      bw.put((uint32_t)(emax + 127), 8);
      uint32_t u[SZ];                          // sequency order, negabinary (R10, R11)
      static_for<0, SZ>([&](auto J) {
        constexpr int j = decltype(J)::value;
        u[j] = to_negabinary(cf[Tab<D>::make_perm().v[j]]);
      });
      const int kmin = 32 - prec;
      int n = 0;                               // coefficients already significant
      for (int kp = 31; kp >= kmin; --kp) {
        // bit plane kp over the sequency order: the planes are visited from the top, so the
        // plane's bit of u[j] is its current top bit -- one funnel shift moves it into the
        // mask, one add drops it (2 instructions per coefficient and plane)
        uint32_t mlo = 0u, mhi = 0u;
#pragma unroll
        for (int j = SZ - 1; j >= 0; --j) {
          if (j >= 32) mhi = __funnelshift_l(u[j], mhi, 1);
          else mlo = __funnelshift_l(u[j], mlo, 1);
          u[j] += u[j];
        }
        const unsigned long long mask = ((unsigned long long)mhi << 32) | mlo;
        bw.put64(mask, n);                     // (i) bits of 0..n-1 verbatim
        while (n < SZ) {                       // (ii) group tests
          const unsigned long long rest = mask >> n;
          bw.put(rest != 0ull ? 1u : 0u, 1);
          if (rest == 0ull) break;
          const int p = n + __ffsll((long long)rest) - 1;   // next significant position
          if (p == SZ - 1) {                   // the last coefficient's 1 is implied
            bw.zeros(p - n);
            n = SZ;
          } else {
            bw.zeros(p - n);
            bw.put(1u, 1);
            n = p + 1;
          }
        }
      }
    }
    bw.flush();
    pos += bits[t];
  }
}

namespace {
template <int D, bool VEC>
struct ZFns {
  static const void *bits() { return (const void *)k_zbits<D, VEC>; }
  static const void *write() { return (const void *)k_zwrite<D, VEC>; }
};
const void *pick_zbits(int D, bool v) {
  if (D == 1) return v ? ZFns<1, true>::bits() : ZFns<1, false>::bits();
  if (D == 2) return v ? ZFns<2, true>::bits() : ZFns<2, false>::bits();
  return v ? ZFns<3, true>::bits() : ZFns<3, false>::bits();
}
const void *pick_zwrite(int D, bool v) {
  if (D == 1) return v ? ZFns<1, true>::write() : ZFns<1, false>::write();
  if (D == 2) return v ? ZFns<2, true>::write() : ZFns<2, false>::write();
  return v ? ZFns<3, true>::write() : ZFns<3, false>::write();
}
}  // namespace

size_t zstream_ws_bytes(int64_t n_pb) {
  const int64_t nc = (n_pb + kScanB - 1) / kScanB;
  return (size_t)n_pb * 4 + (size_t)nc * 8 + 256;
}

// lengths + scan; *d_total receives the stream length in bits
int launch_zstream_bits(const float *x, const Geo &g, int sm_count, const Params *prm, void *ws,
                        unsigned long long *d_total, cudaStream_t st) {
  uint32_t *bits = (uint32_t *)ws;
  unsigned long long *csum = (unsigned long long *)((char *)ws + (((size_t)g.n_pb * 4 + 255) & ~(size_t)255));
  const int64_t nc = (g.n_pb + kScanB - 1) / kScanB;
  int64_t ctas = (g.n_pb + 255) / 256;
  if (ctas > (int64_t)sm_count * 8) ctas = (int64_t)sm_count * 8;
  Geo gg = g;
  void *a1[] = {(void *)&x, (void *)&gg, (void *)&prm, (void *)&bits};
  if (cudaLaunchKernel(pick_zbits(g.ndims, g.vec != 0), dim3((unsigned)ctas), dim3(256), a1, 0, st) != cudaSuccess)
    return SEL_ECUDA;
  k_scan_sum<<<(unsigned)nc, 256, 0, st>>>(bits, g.n_pb, csum);
  k_scan_top<<<1, 1024, 0, st>>>(csum, (int)nc, d_total);
  return cudaGetLastError() == cudaSuccess ? SEL_OK : SEL_ECUDA;
}

int launch_zstream_write(const float *x, const Geo &g, const Params *prm, void *ws, uint32_t *out, cudaStream_t st) {
  const uint32_t *bits = (const uint32_t *)ws;
  const unsigned long long *cbase =
      (const unsigned long long *)((char *)ws + (((size_t)g.n_pb * 4 + 255) & ~(size_t)255));
  const int64_t nc = (g.n_pb + kScanB - 1) / kScanB;
  Geo gg = g;
  void *a[] = {(void *)&x, (void *)&gg, (void *)&prm, (void *)&bits, (void *)&cbase, (void *)&out};
  return cudaLaunchKernel(pick_zwrite(g.ndims, g.vec != 0), dim3((unsigned)nc), dim3(256), a, 0, st) == cudaSuccess
             ? SEL_OK
             : SEL_ECUDA;
}

}  // namespace sel
