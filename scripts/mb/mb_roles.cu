// Microbenchmark (developer tool): 3D tile consumer with the SZ and ZFP halves on different
// warps (ROLE split) on a resident smem tile.  Variants: V=0 8 warps both halves (the
// committed consumer), V=1 8 SZ warps only, V=2 8 ZFP warps only, V=3 8 SZ + 8 ZFP warps
// with setmaxnreg (SZ warpgroups dec, ZFP warpgroups inc).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false \
//        --expt-relaxed-constexpr -I include -o /tmp/mb_roles scripts/mb/mb_roles.cu
#include <cstdio>
#include <cmath>
#include "../../paper_1806_08901_b200/csrc/sel_tile_common.cuh"
using namespace sel;

#ifndef RZ
#define RZ 144
#endif
#ifndef RZ4
#define RZ4 200
#endif
#ifndef RS4
#define RS4 72
#endif
#ifndef RS
#define RS 72
#endif

template <int V>
constexpr int nthreads() { return V == 3 ? 512 + 128 : V == 4 ? 512 : 256; }

template <int V>
__global__ void __launch_bounds__(nthreads<V>(), 1)
    k_mb(int iters, float r_f, int minexp, float amp, float noise, unsigned int *gh, unsigned long long *sink) {
  using Cfg = TileCfg<3>;
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
  if constexpr (V == 3) {
    if (warp >= 16) {          // helper warpgroup: idle
      asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
      return;
    }
    if (warp < 8) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(RS));
      for (int it = 0; it < iters; ++it) {
        uint64_t tb; double te;
        tile_consume<3, false, unsigned int, 1>(S, 1 + (it & 1), 1, 1, tg, warp, lane, true, r_f, minexp, win, gh, ovf, nd, tb, te);
      }
    } else {
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(RZ));
      for (int it = 0; it < iters; ++it) {
        uint64_t tb; double te;
        tile_consume<3, false, unsigned int, 2>(S, 1 + (it & 1), 1, 1, tg, warp - 8, lane, true, r_f, minexp, win, gh, ovf, nd, tb, te);
        acc += tb; eacc += te;
      }
    }
  } else if constexpr (V == 4) {   // warps 0-3 helpers, 4-7 SZ (2 block rows each), 8-15 ZFP
    if (warp < 4) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
      return;
    }
    if (warp < 8) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(RS4));
      for (int it = 0; it < iters; ++it) {
        uint64_t tb; double te;
        tile_consume<3, false, unsigned int, 1>(S, 1 + (it & 1), 1, 1, tg, warp - 4, lane, true, r_f, minexp, win, gh, ovf, nd, tb, te);
        tile_consume<3, false, unsigned int, 1>(S, 1 + (it & 1), 1, 1, tg, warp, lane, true, r_f, minexp, win, gh, ovf, nd, tb, te);
      }
    } else {
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(RZ4));
      for (int it = 0; it < iters; ++it) {
        uint64_t tb; double te;
        tile_consume<3, false, unsigned int, 2>(S, 1 + (it & 1), 1, 1, tg, warp - 8, lane, true, r_f, minexp, win, gh, ovf, nd, tb, te);
        acc += tb; eacc += te;
      }
    }
  } else {
    for (int it = 0; it < iters; ++it) {
      uint64_t tb; double te;
      tile_consume<3, false, unsigned int, V>(S, 1 + (it & 1), 1, 1, tg, warp, lane, true, r_f, minexp, win, gh, ovf, nd, tb, te);
      acc += tb; eacc += te;
    }
  }
  if (acc == 0x1234567ull) sink[0] = (unsigned long long)eacc + ovf;   // keep the work alive
  sink[1 + blockIdx.x * blockDim.x + threadIdx.x] = acc + ovf;
}

template <int V>
void run(float r_f, int minexp, float amp, float noise, const char *label) {
  using Cfg = TileCfg<3>;
  const size_t smem = (size_t)Cfg::STAGE_FLOATS * 4 + Cfg::HIST_WORDS * 4;
  cudaFuncSetAttribute(k_mb<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned int *gh; unsigned long long *sink;
  cudaMalloc(&gh, 70000 * 4);
  cudaMalloc(&sink, (1 + sms * 1024) * 8);
  const int iters = 200;
  k_mb<V><<<sms, nthreads<V>(), smem>>>(10, r_f, minexp, amp, noise, gh, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_mb<V><<<sms, nthreads<V>(), smem>>>(iters, r_f, minexp, amp, noise, gh, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double vals = (double)sms * 8 * 32 * 64 * iters;
  fflush(stdout); printf("V=%d %-22s: %.3f ms, %.1f Gvalues/s = %.0f GB/s of float32 (%s)\n", V, label, ms,
         vals / ms / 1e6, vals * 4 / ms / 1e6, cudaGetErrorString(cudaGetLastError())); fflush(stdout);
}

int main() {
  run<0>(2000.f, -12, 1.0f, 1e-3f, "both, 8 warps smooth");
  run<1>(2000.f, -12, 1.0f, 1e-3f, "SZ only, 8 warps");
  run<2>(2000.f, -12, 1.0f, 1e-3f, "ZFP only, 8 warps");
  run<4>(2000.f, -12, 1.0f, 1e-3f, "4 SZ + 8 ZFP warps");
  run<3>(2000.f, -12, 1.0f, 1e-3f, "8 SZ + 8 ZFP warps");
  run<0>(2000.f, -12, 1.0f, 0.05f, "both, noise +-100");
  run<4>(2000.f, -12, 1.0f, 0.05f, "4+8, noise +-100");
  run<3>(2000.f, -12, 1.0f, 0.05f, "8+8, noise +-100");
  return 0;
}
