// Microbenchmark (developer tool): the 3D tile consumer (8 warps, resident tile) with the
// k_batch background traffic switched on one at a time: BG bit 0 = a producer warp
// bulk-copying 87 KB global -> a second smem stage back to back; bit 1 = two warps
// streaming LDG.128 min/max over a large global buffer.
#include <cstdio>
#include <cmath>
#include "../../paper_1806_08901_b200/csrc/sel_tile_common.cuh"
using namespace sel;

__device__ __forceinline__ void bulk_ld(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int BG>
__global__ void __launch_bounds__(384, 1)
    k_mb(int iters, float r_f, int minexp, const float *gsrc, size_t gn, unsigned int *gh, unsigned long long *sink, TileGeo tg, int3 tc) {
  using Cfg = TileCfg<3>;
  extern __shared__ __align__(128) float sm[];
  float *S = sm;
  float *S2 = sm + Cfg::STAGE_FLOATS;
  unsigned int *win = reinterpret_cast<unsigned int *>(sm + 2 * Cfg::STAGE_FLOATS);
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < Cfg::STAGE_FLOATS; i += blockDim.x) {
    const float t = (float)i;
    unsigned h = (unsigned)i * 2654435761u + blockIdx.x * 40503u;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    const float u = (float)(h & 0xffffff) / 16777216.0f - 0.5f;
    S[i] = sinf(t * 0.013f) + 0.5f * cosf(t * 0.0071f + (float)blockIdx.x) + 1e-3f * u;
  }
  for (int i = threadIdx.x; i < Cfg::HIST_WORDS; i += blockDim.x) win[i] = 0u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); stop = 0; }
  __syncthreads();
  if (warp == 8) {          // producer
    if ((BG & 1) && lane == 0) {
      uint32_t ph = 0;
      size_t off = (size_t)blockIdx.x * 1048576;
      while (!stop) {
        mbar_arrive_expect_tx(&bar, Cfg::STAGE_BYTES);
        bulk_ld(S2, gsrc + off, Cfg::STAGE_BYTES, &bar);
        mbar_wait_sleep(&bar, ph);
        ph ^= 1u;
        off += Cfg::STAGE_BYTES / 4 * 148;
        if (off + Cfg::STAGE_BYTES / 4 >= gn) off = (size_t)blockIdx.x * 1048576;
      }
    }
    return;
  }
  if (warp == 9) return;
  if (warp >= 10) {         // range warps
    if (BG & 2) {
      float mn = INFINITY, mx = -INFINITY;
      const float4 *src = reinterpret_cast<const float4 *>(gsrc);
      size_t i = ((size_t)blockIdx.x * 2 + (warp - 10)) * 65536 + lane;
      while (!stop) {
        float4 q[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) q[k] = __ldg(src + i + k * 32);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          mn = fminf(fminf(mn, q[k].x), fminf(q[k].y, fminf(q[k].z, q[k].w)));
          mx = fmaxf(fmaxf(mx, q[k].x), fmaxf(q[k].y, fmaxf(q[k].z, q[k].w)));
        }
        i += 16 * 32 * 296;
        if (i + 16 * 32 >= gn / 4) i = ((size_t)blockIdx.x * 2 + (warp - 10)) * 65536 + lane;
      }
      if (mn == 123.f) sink[0] = (unsigned long long)mx;
    }
    return;
  }
  DebugPtrs nd{};
  unsigned int ovf = 0;
  unsigned long long acc = 0;
  double eacc = 0.0;
  for (int it = 0; it < iters; ++it) {
    uint64_t tb; double te;
    tile_consume<3, false, unsigned int>(S, tc.x + (it & 1), tc.y, tc.z, tg, warp, lane, true, r_f, minexp, win, gh, ovf, nd, tb, te);
    acc += tb; eacc += te;
  }
  asm volatile("bar.sync 1, 256;");
  if (threadIdx.x == 0) stop = 1;
  if (acc == 0x1234567ull) sink[0] = (unsigned long long)eacc + ovf;
  sink[1 + blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int BG>
void run(const float *gsrc, size_t gn, const char *label) {
  using Cfg = TileCfg<3>;
  const size_t smem = (size_t)2 * Cfg::STAGE_FLOATS * 4 + Cfg::HIST_WORDS * 4;
  cudaFuncSetAttribute(k_mb<BG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned int *gh; unsigned long long *sink;
  cudaMalloc(&gh, 70000 * 4);
  cudaMalloc(&sink, (1 + 148 * 384) * 8);
  const int iters = 200;
  TileGeo tg;
  tg.n[0] = 1 << 20; tg.n[1] = 1 << 20; tg.n[2] = 1 << 20;
  tg.nb[0] = 1 << 18; tg.nb[1] = 1 << 18; tg.nb[2] = 1 << 18;
  tg.ntj = 1 << 10; tg.ntk = 1 << 10; tg.ntasks = 1 << 20;
  const int3 tc = make_int3(1, 1, 1);
  k_mb<BG><<<148, 384, smem>>>(10, 2000.f, -12, gsrc, gn, gh, sink, tg, tc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_mb<BG><<<148, 384, smem>>>(iters, 2000.f, -12, gsrc, gn, gh, sink, tg, tc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double vals = (double)148 * 8 * 32 * 64 * iters;
  printf("BG=%d %-34s: %.3f ms, %.0f GB/s of float32, %.3f cycles/value/SM @1.965 GHz (%s)\n", BG, label, ms,
         vals * 4 / ms / 1e6, ms * 1e-3 * 1.965e9 * 148 / vals, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

int main() {
  size_t gn = (size_t)1 << 30;     // 4 GiB of floats
  float *g;
  cudaMalloc(&g, gn * 4);
  cudaMemset(g, 0, gn * 4);
  run<0>(g, gn, "consumers alone");
  run<1>(g, gn, "+ bulk copies into stage 2");
  run<2>(g, gn, "+ 2 LDG range warps");
  run<3>(g, gn, "+ both");
  return 0;
}
