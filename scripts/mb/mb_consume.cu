// Microbenchmark (developer tool): the tile consumer's compute alone -- every consumer
// warp runs tile_consume on a resident, pre-filled smem tile in a loop (no producer, no
// TMA, no task scheduling), one CTA per SM.  Gives the compute ceiling of the T tasks.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false \
//        --expt-relaxed-constexpr -I include -o /tmp/mb_consume scripts/mb/mb_consume.cu -lcuda
#include <cstdio>
#include <cmath>
#include "../../paper_1806_08901_b200/csrc/sel_tile_common.cuh"
using namespace sel;

template <int D>
__global__ void __launch_bounds__(TileCfg<D>::CW * 32, 1)
    k_mb(int iters, float r_f, int minexp, float amp, float noise, unsigned int *gh, unsigned long long *sink) {
  using Cfg = TileCfg<D>;
  extern __shared__ float sm[];
  float *S = sm;
  unsigned int *win = reinterpret_cast<unsigned int *>(sm + Cfg::STAGE_FLOATS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < Cfg::STAGE_FLOATS; i += blockDim.x) {
    const float t = (float)i;
    unsigned h = (unsigned)i * 2654435761u + blockIdx.x * 40503u;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    const float u = (float)(h & 0xffffff) / 16777216.0f - 0.5f;
    S[i] = amp * (sinf(t * 0.013f) + 0.5f * cosf(t * 0.0071f + (float)blockIdx.x)) + noise * u;
  }
  for (int i = threadIdx.x; i < Cfg::HIST_WORDS; i += blockDim.x) win[i] = 0u;
  __syncthreads();
  TileGeo tg;
  tg.n[0] = 1 << 20; tg.n[1] = 1 << 20; tg.n[2] = 1 << 20;
  tg.nb[0] = 1 << 18; tg.nb[1] = 1 << 18; tg.nb[2] = 1 << 18;
  tg.ntj = 1 << 10; tg.ntk = 1 << 10; tg.ntasks = 1 << 20;
  DebugPtrs nd{};
  unsigned int ovf = 0;
  unsigned long long acc = 0;
  double eacc = 0.0;
  for (int it = 0; it < iters; ++it) {
    uint64_t tb; double te;
    tile_consume<D, false, unsigned int>(S, 1 + (it & 1), 1, 1, tg, warp, lane, true, r_f, minexp, win, gh,
                                         ovf, nd, tb, te);
    acc += tb;
    eacc += te;
  }
  if (acc == 0x1234567ull) sink[0] = (unsigned long long)eacc + ovf;   // keep the work alive
  sink[1 + blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int D>
void run(float r_f, int minexp, float amp, float noise, const char *label) {
  using Cfg = TileCfg<D>;
  const size_t smem = (size_t)Cfg::STAGE_FLOATS * 4 + Cfg::HIST_WORDS * 4;
  cudaFuncSetAttribute(k_mb<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned int *gh; unsigned long long *sink;
  cudaMalloc(&gh, 70000 * 4);
  cudaMalloc(&sink, (1 + sms * Cfg::CW * 32) * 8);
  const int iters = D == 3 ? 200 : 2000;
  k_mb<D><<<sms, Cfg::CW * 32, smem>>>(10, r_f, minexp, amp, noise, gh, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_mb<D><<<sms, Cfg::CW * 32, smem>>>(iters, r_f, minexp, amp, noise, gh, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double vals = (double)sms * Cfg::CW * 32 * (D == 3 ? 64 : 16) * iters;
  printf("D=%d %-28s CW=%d: %.3f ms, %.1f Gvalues/s = %.0f GB/s of float32 (%s)\n", D, label, Cfg::CW, ms,
         vals / ms / 1e6, vals * 4 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  // r_f: codes of a smooth field (spread ~ +-100) and of a rough one (~ +-3000)
  // codes of noise of amplitude a: |code| ~ a * r_f (spread over +- a r_f bins)
  run<2>(2000.f, -12, 1.0f, 1e-3f, "smooth");
  run<2>(2000.f, -12, 1.0f, 0.05f, "noise +-100 codes");
  run<2>(2000.f, -12, 1.0f, 0.5f, "noise +-1000 codes");
  run<2>(2000.f, -12, 1.0f, 2.0f, "noise +-4000 codes");
  run<3>(2000.f, -12, 1.0f, 1e-3f, "smooth");
  run<3>(2000.f, -12, 1.0f, 0.05f, "noise +-100 codes");
  run<3>(2000.f, -12, 1.0f, 0.5f, "noise +-1000 codes");
  return 0;
}
