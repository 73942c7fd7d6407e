// Issue-rate microbenchmark for the instructions the attend kernels lean on (B200).
// Each kernel: 148*8 CTAs x 256 threads, 8 independent chains per thread, N iterations.
#include <cstdio>
#include <cuda_fp16.h>
#define N 4096
__global__ void k_ffma(float *o, float a) {
  float x[8]; for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int n = 0; n < N; ++n)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, 0.5f);
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i]; if (s == 1.2345f) o[0] = s;
}
__global__ void k_fhfma(float *o, unsigned b) {
  float x[8]; for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  unsigned a = threadIdx.x * 0x10001u;
  for (int n = 0; n < N; ++n)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("{.reg .b16 x0,x1,y0,y1; mov.b32 {x0,x1}, %1; mov.b32 {y0,y1}, %2; fma.rn.f32.f16 %0, x0, y0, %0;}" : "+f"(x[i]) : "r"(a), "r"(b));
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i]; if (s == 1.2345f) o[0] = s;
}
__global__ void k_ffma2(float *o, float a) {
  unsigned long long x[8]; for (int i = 0; i < 8; ++i) { float2 f = make_float2(threadIdx.x + i, i); x[i] = *(unsigned long long *)&f; }
  float2 af = make_float2(a, a); unsigned long long av = *(unsigned long long *)&af;
  for (int n = 0; n < N; ++n)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(x[i]) : "l"(av));
  float s = 0; for (int i = 0; i < 8; ++i) s += ((float2 *)&x[i])->x; if (s == 1.2345f) o[0] = s;
}
__global__ void k_mufu(float *o, float a) {
  float x[8]; for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int n = 0; n < N; ++n)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("sin.approx.f32 %0, %0;" : "+f"(x[i]));
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i]; if (s == 1.2345f) o[0] = s;
}
__global__ void k_hmma(float *o, unsigned b) {
  float d[4][4] = {}; unsigned a = threadIdx.x * 0x10001u;
  for (int n = 0; n < N / 4; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};"
                   : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3]) : "r"(a), "r"(b));
  float s = 0; for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][3]; if (s == 1.2345f) o[0] = s;
}
__global__ void k_imma(float *o, unsigned b) {
  int d[4][4] = {}; unsigned a = threadIdx.x * 0x01010101u;
  for (int n = 0; n < N / 4; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};"
                   : "+r"(d[i][0]), "+r"(d[i][1]), "+r"(d[i][2]), "+r"(d[i][3]) : "r"(a), "r"(b));
  int s = 0; for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][3]; if (s == 12345) o[0] = s;
}
__global__ void k_lop(float *o, unsigned b) {
  unsigned x[8]; for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int n = 0; n < N; ++n)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("lop3.b32 %0, %0, %1, 0x3c, 0x6a;" : "+r"(x[i]) : "r"(b));
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += x[i]; if (s == 12345) o[0] = s;
}
__global__ void k_shf(float *o, unsigned b) {
  unsigned x[8]; for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int n = 0; n < N; ++n)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("shf.r.wrap.b32 %0, %0, %1, %1;" : "+r"(x[i]) : "r"(b));
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += x[i]; if (s == 12345) o[0] = s;
}
__global__ void k_f2fp(float *o, float a) {
  float x[8]; for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  unsigned acc = 0;
  for (int n = 0; n < N; ++n)
#pragma unroll
    for (int i = 0; i < 8; i += 2) { unsigned r; asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[i]), "f"(x[i+1])); acc ^= r; }
  if (acc == 12345) o[0] = acc;
}
template <typename K, typename A>
void run(const char *name, K k, A arg, double ops_per_iter_per_thread) {
  float *o; cudaMalloc(&o, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<148 * 8, 256>>>(o, arg);
  cudaEventRecord(e0);
  k<<<148 * 8, 256>>>(o, arg);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double warp_instr = 148.0 * 8 * 8 * N * ops_per_iter_per_thread;   // warps * per-warp instructions
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-8s %8.3f ms  %6.2f warp-instr/clk/SM (at %d MHz nominal)\n", name, ms, warp_instr / 148 / cyc, clk / 1000);
}
int main() {
  run("FFMA", k_ffma, 1.0001f, 8);
  run("FHFMA", k_fhfma, 0x3c003c00u, 8);
  run("FFMA2", k_ffma2, 1.0001f, 8);
  run("MUFU", k_mufu, 1.f, 8);
  run("LOP3", k_lop, 7u, 8);
  run("SHF", k_shf, 7u, 8);
  run("F2FP", k_f2fp, 1.f, 4);
  run("HMMA", k_hmma, 0x3c003c00u, 1);
  run("IMMA", k_imma, 0x01010101u, 1);
  return 0;
}
