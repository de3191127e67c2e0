// Microbenchmark: warp-instruction throughput per SM for the instruction
// classes of the scan inner loop (B200, sm_100a). Each kernel runs 8
// independent chains per thread; full occupancy; events around many iters.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
#define CHAINS 8

__global__ void k_ffma(float* o, float a, float b) {
  float x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = __fmaf_rn(x[c], a, b);
  float s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 1.2345f) o[0] = s;
}
__global__ void k_fadd(float* o, float a, float b) {
  float x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = __fadd_rn(x[c], a);
  float s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 1.2345f) o[0] = s;
}
__global__ void k_ffma2(float* o, float a, float b) {
  float2 x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = make_float2(threadIdx.x * 1e-3f + c, c);
  float2 aa = make_float2(a, a), bb = make_float2(b, b);
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = __ffma2_rn(x[c], aa, bb);
  float s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c].x + x[c].y;
  if (s == 1.2345f) o[0] = s;
}
__global__ void k_fadd2(float* o, float a, float b) {
  float2 x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = make_float2(threadIdx.x * 1e-3f + c, c);
  float2 aa = make_float2(a, b);
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = __fadd2_rn(x[c], aa);
  float s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c].x + x[c].y;
  if (s == 1.2345f) o[0] = s;
}
// FSETP-heavy: compare and predicated add (per chain: 1 FSETP + 1 @P FADD)
__global__ void k_fsetp(float* o, float a, float b) {
  float x[CHAINS], y[CHAINS];
  for (int c = 0; c < CHAINS; ++c) { x[c] = threadIdx.x * 1e-3f + c; y[c] = 0; }
  unsigned f = 0;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      asm volatile("{.reg .pred p; setp.gt.f32 p, %1, %2; @p add.rn.f32 %0, %0, %3;}" : "+f"(y[c]) : "f"(x[c]), "f"(a), "f"(b));
    }
  float s = 0; for (int c = 0; c < CHAINS; ++c) s += y[c];
  if (s == 1.2345f) o[0] = s + f;
}
// pure FSETP accumulate into predicate (2 FSETP per chain-iter)
__global__ void k_fsetp_only(float* o, float a, float b) {
  float x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3f + c;
  unsigned f = 0;
  for (int i = 0; i < ITERS; ++i) {
    asm volatile("{.reg .pred p; setp.ne.u32 p, %0, 0;\n\t"
      "setp.gt.or.f32 p, %1, %9, p; setp.gt.or.f32 p, %2, %9, p; setp.gt.or.f32 p, %3, %9, p; setp.gt.or.f32 p, %4, %9, p;\n\t"
      "setp.gt.or.f32 p, %5, %9, p; setp.gt.or.f32 p, %6, %9, p; setp.gt.or.f32 p, %7, %9, p; setp.gt.or.f32 p, %8, %9, p;\n\t"
      "selp.u32 %0, 1, 0, p;}" : "+r"(f) : "f"(x[0]),"f"(x[1]),"f"(x[2]),"f"(x[3]),"f"(x[4]),"f"(x[5]),"f"(x[6]),"f"(x[7]),"f"(a));
  }
  if (f == 12345) o[0] = f;
}
__global__ void k_iadd(float* o, float a, float b) {
  int x[CHAINS]; int ai = __float_as_int(a);
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) asm volatile("add.s32 %0, %0, %1;" : "+r"(x[c]) : "r"(ai));
  int s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345) o[0] = s;
}

typedef void (*KF)(float*, float, float);
int main() {
  float* d; cudaMalloc(&d, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  struct { const char* n; KF f; double instr_per_chain_iter; } ks[] = {
    {"FFMA", k_ffma, 1}, {"FADD", k_fadd, 1}, {"FFMA2", k_ffma2, 1}, {"FADD2", k_fadd2, 1},
    {"FSETP+@P FADD", k_fsetp, 2}, {"FSETP.OR only", k_fsetp_only, 1}, {"IADD", k_iadd, 1}};
  int threads = 1024, blocks = sms * 2;
  for (auto& k : ks) {
    k.f<<<blocks, threads>>>(d, 1.0001f, 0.5f);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k.f<<<blocks, threads>>>(d, 1.0001f, 0.5f);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double warp_instr = 5.0 * blocks * (threads / 32) * (double)ITERS * CHAINS * k.instr_per_chain_iter;
    double per_sm_per_ns = warp_instr / sms / (ms * 1e6);
    printf("%-16s %8.3f ms  %.3f warp-instr/ns/SM  (= %.2f per clk at %.0f MHz max)\n", k.n, ms, per_sm_per_ns,
           per_sm_per_ns / (clk / 1e6), clk / 1e3);
  }
  return 0;
}
