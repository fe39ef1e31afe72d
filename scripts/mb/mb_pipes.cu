// Microbenchmark (developer tool): issue rate of the integer ops of the ZFP lift on sm_100a,
// 8 warps per SM (2 per SMSP), 16 independent chains per thread.  MODE 0: add.s32 only;
// 1: mad.lo.s32 (x*one + y, one is a run-time 1) only; 2: alternating add / mad; 3: shr only;
// 4: add, shr, mad triples (the lift's mix with the adds on the FMA pipe); 5: add, shr, add.
#include <cstdio>
template <int MODE>
__global__ void __launch_bounds__(256, 1) k(int iters, int one, int *out) {
  int a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x + i;
  int b = blockIdx.x + 3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (MODE == 0) { asm volatile("add.s32 %0, %0, %1;" : "+r"(a[i]) : "r"(b)); }
        if (MODE == 1) { asm volatile("mad.lo.s32 %0, %1, %2, %0;" : "+r"(a[i]) : "r"(b), "r"(one)); }
        if (MODE == 2) { if (i & 1) asm volatile("add.s32 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
                         else asm volatile("mad.lo.s32 %0, %1, %2, %0;" : "+r"(a[i]) : "r"(b), "r"(one)); }
        if (MODE == 3) { asm volatile("shr.s32 %0, %0, 1;" : "+r"(a[i])); }
        if (MODE == 4) { asm volatile("add.s32 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
                         asm volatile("shr.s32 %0, %0, 1;" : "+r"(a[i]));
                         asm volatile("mad.lo.s32 %0, %1, %2, %0;" : "+r"(a[i]) : "r"(b), "r"(one)); }
        if (MODE == 5) { asm volatile("add.s32 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
                         asm volatile("shr.s32 %0, %0, 1;" : "+r"(a[i]));
                         asm volatile("add.s32 %0, %0, %1;" : "+r"(a[i]) : "r"(b)); }
        if (MODE == 6) { asm volatile("mad.lo.s32 %0, %1, %2, %0;" : "+r"(a[i]) : "r"(b), "r"(one));
                         asm volatile("shr.s32 %0, %0, 1;" : "+r"(a[i]));
                         asm volatile("mad.lo.s32 %0, %1, %2, %0;" : "+r"(a[i]) : "r"(b), "r"(one)); }
      }
    }
  }
  int s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= a[i];
  out[blockIdx.x * 256 + threadIdx.x] = s;
}
template <int MODE>
void run(const char *label, int per) {
  int *out; cudaMalloc(&out, 148 * 256 * 4);
  k<MODE><<<148, 256>>>(10, 1, out);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  cudaEventRecord(e0);
  k<MODE><<<148, 256>>>(iters, 1, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double winstr = (double)iters * 64 * per * 2;   // per SMSP: 2 warps
  printf("MODE %d %-28s: %.3f ms, %.3f warp-instr/cycle/SMSP @1.965 GHz\n", MODE, label, ms, winstr / (ms * 1e-3 * 1.965e9));
}
int main() {
  run<0>("add", 1); run<1>("mad.lo (x*1+y)", 1); run<2>("add / mad alternating", 1); run<3>("shr", 1);
  run<4>("add, shr, mad", 3); run<5>("add, shr, add", 3); run<6>("mad, shr, mad", 3);
  return 0;
}
