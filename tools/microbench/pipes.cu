// Pipe-throughput microbenchmark for the ALU roofline denominator.
// Measures, full-chip, sustained warp-instruction throughput for the instruction
// classes the assess kernel issues: FFMA (reg), FADD, FFMA2 (f32x2), DFMA, LDS.32/64, MUFU.RSQ.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_ffma(float* out, float a, float b) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b + x[(i + 3) & 7] * 0.0f);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.f) out[0] = s;
}

// pure FFMA chains, 3 distinct registers
__global__ void k_ffma3(float* out, float a, float b) {
  float x[8], y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 1e-3f + i; y[i] = a + i; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], y[i], x[(i + 1) & 7]);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_fadd(float* out, float a) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = x[i] + x[(i + 1) & 7];
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
  unsigned long long x[8], y;
  {
    float2 t = make_float2(a, b);
    y = *reinterpret_cast<unsigned long long*>(&t);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) { float2 t = make_float2(threadIdx.x * 1e-3f + i, i); x[i] = *reinterpret_cast<unsigned long long*>(&t); }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(y), "l"(x[(i + 1) & 7]));
  }
  float s = 0; for (int i = 0; i < 8; ++i) { float2 t = *reinterpret_cast<float2*>(&x[i]); s += t.x + t.y; }
  if (s == 12345.f) out[0] = s;
}

__global__ void k_dfma(float* out, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, x[(i + 1) & 7]);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0) out[0] = (float)s;
}

__global__ void k_rsq(float* out) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i + 1;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = rsqrtf(x[i]);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_lds32(float* out) {
  __shared__ float sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
  __syncthreads();
  float acc[8] = {0};
  int base = threadIdx.x;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] += sm[(base + i * 32 + it) & 4095];
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_lds64(float* out) {
  __shared__ float2 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_float2(i, i);
  __syncthreads();
  float acc[8] = {0};
  int base = threadIdx.x;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { float2 v = sm[(base + i * 32 + it) & 2047]; acc[i] += v.x + v.y; }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.f) out[0] = s;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("{\"sms\": %d, \"clock_khz_attr\": %d}\n", nsm, clk);
  float* out; CK(cudaMalloc(&out, 16));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 256, blocks = nsm * 8;
  struct R { const char* name; double ops_per_thread; double insts_per_thread; };
  auto run = [&](const char* name, auto launch, double ops_per_thread, double insts_per_thread) {
    for (int w = 0; w < 2; ++w) launch();
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double s = ms * 1e-3 / reps;
    double thr = (double)blocks * threads;
    double ops = thr * ops_per_thread / s;
    double warp_insts = thr / 32 * insts_per_thread / s;
    printf("{\"op\": \"%s\", \"ms\": %.4f, \"Gops_per_s\": %.1f, \"warp_inst_per_s_per_sm\": %.4g}\n",
           name, s * 1e3, ops / 1e9, warp_insts / nsm);
    return 0;
  };
  run("ffma_fp32 (1 FMA = 2 flop; counts FMA)", [&] { k_ffma<<<blocks, threads>>>(out, 1.0001f, 1e-7f); }, 8.0 * ITERS, 8.0 * ITERS);
  run("ffma3_fp32 (3 distinct regs)", [&] { k_ffma3<<<blocks, threads>>>(out, 1.0001f, 1e-7f); }, 8.0 * ITERS, 8.0 * ITERS);
  run("fadd_fp32", [&] { k_fadd<<<blocks, threads>>>(out, 1.0f); }, 8.0 * ITERS, 8.0 * ITERS);
  run("ffma2_f32x2 (counts 2 FMA per inst)", [&] { k_ffma2<<<blocks, threads>>>(out, 1.0001f, 1e-7f); }, 16.0 * ITERS, 8.0 * ITERS);
  run("dfma_fp64", [&] { k_dfma<<<blocks, threads>>>(out, 1.0000001, 1e-9); }, 8.0 * ITERS / 4, 8.0 * ITERS / 4);
  run("mufu_rsq", [&] { k_rsq<<<blocks, threads>>>(out); }, 8.0 * ITERS / 4, 8.0 * ITERS / 4);
  run("lds32 (+fadd)", [&] { k_lds32<<<blocks, threads>>>(out); }, 8.0 * ITERS / 4, 8.0 * ITERS / 4);
  run("lds64 (+2 fadd)", [&] { k_lds64<<<blocks, threads>>>(out); }, 8.0 * ITERS / 4, 8.0 * ITERS / 4);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}
