// MUFU.EX2 / F2FP / FFMA2 issue rates per SM on this GPU (clock64 cycles).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_rate mufu_rate.cu
#include <cstdio>
#include <cstdint>
__global__ void ex2_kernel(float* out, long long* cyc, int iters) {
  float a = threadIdx.x * 1e-3f, b = a + 0.5f, c = a + 0.25f, d = a + 0.125f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(c));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(d));
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}
__global__ void f2fp_kernel(float* out, long long* cyc, int iters) {
  float a = threadIdx.x * 1e-3f, b = a + 0.5f;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r0, r1, r2, r3;
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r0) : "f"(a), "f"(b));
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r1) : "f"(b), "f"(a));
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r2) : "f"(a), "f"(a));
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r3) : "f"(b), "f"(b));
    acc ^= r0 ^ r1 ^ r2 ^ r3;
    a += 1e-7f;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}
// packed half-precision ex2: two results per instruction if MUFU runs it as one op
__global__ void ex2h2_kernel(float* out, long long* cyc, int iters, int bf) {
  uint32_t a = 0x3c003c00u + threadIdx.x, b = a ^ 0x10001u, c = a ^ 0x20002u, d = a ^ 0x30003u;
  __syncthreads();
  long long t0 = clock64();
  if (bf) {
    for (int i = 0; i < iters; ++i) {
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a));
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(b));
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(c));
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(d));
    }
  } else {
    for (int i = 0; i < iters; ++i) {
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a));
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(b));
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(c));
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(d));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(a ^ b ^ c ^ d);
}
int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  for (int threads : {128, 256, 512, 1024}) {
    for (int k = 0; k < 2; ++k) {
      if (k == 0) ex2_kernel<<<148, threads>>>(out, cyc, iters);
      else f2fp_kernel<<<148, threads>>>(out, cyc, iters);
      long long h[148];
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double ops = 4.0 * iters * threads;
      printf("%s threads/SM %4d: %.2f ops/clk/SM\n", k ? "cvt.f16x2" : "ex2", threads, ops / h[0]);
    }
  }
  for (int threads : {256, 512, 1024})
    for (int bf = 0; bf < 2; ++bf) {
      ex2h2_kernel<<<148, threads>>>(out, cyc, iters, bf);
      long long h[148];
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      printf("%s threads/SM %4d: %.2f instr/clk/SM (x2 values)\n",
             bf ? "ex2.bf16x2" : "ex2.f16x2", threads, 4.0 * iters * threads / h[0]);
    }
  return 0;
}
