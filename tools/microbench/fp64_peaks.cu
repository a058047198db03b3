// Microbenchmark: FP64 DMMA (mma.sync m8n8k4 f64) vs DFMA throughput, grid-barrier
// latency and streaming-read bandwidth on sm_100a. Used once to pick the ADMM kernel
// design.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int i = 0; i < 8; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0; for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8];
  for (int i = 0; i < 8; i++) c[i] = i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) c[i] = fma(a, c[i], b);
  }
  double s = 0; for (int i = 0; i < 8; i++) s += c[i];
  if (s == 12345.678) out[0] = s;
}
__device__ unsigned g_count, g_gen;
__global__ void barrier_loop(int iters) {
  for (int it = 0; it < iters; it++) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned gen;
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(gen) : "l"(&g_gen));
      unsigned prev = atomicAdd(&g_count, 1);
      if (prev == gridDim.x - 1) {
        g_count = 0;
        asm volatile("st.release.gpu.u32 [%0], %1;" :: "l"(&g_gen), "r"(gen + 1));
      } else {
        unsigned cur;
        do { asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(&g_gen)); } while (cur == gen);
      }
    }
    __syncthreads();
  }
}
__global__ void stream_read(const double2* __restrict__ x, size_t n2, double* out) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride * 4) {
    double2 v0 = __ldcs(x + i);
    double2 v1 = (i + stride < n2) ? __ldcs(x + i + stride) : make_double2(0,0);
    double2 v2 = (i + 2*stride < n2) ? __ldcs(x + i + 2*stride) : make_double2(0,0);
    double2 v3 = (i + 3*stride < n2) ? __ldcs(x + i + 3*stride) : make_double2(0,0);
    acc += v0.x + v1.x + v2.x + v3.x + v0.y + v1.y + v2.y + v3.y;
  }
  if (acc == 1.2345) out[0] = acc;
}
int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int l2; CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("SMs %d L2 %d MB clock %d MHz\n", sms, l2 >> 20, clk / 1000);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    int iters = 20000; int blocks = sms * 2;
    dmma_loop<<<blocks, warps * 32>>>(out, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dmma_loop<<<blocks, warps * 32>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)blocks * warps;
    printf("DMMA warps/blk %2d x2 blk/SM: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
    dfma_loop<<<blocks, warps * 32>>>(out, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dfma_loop<<<blocks, warps * 32>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 8 * iters * (double)blocks * warps * 32;
    printf("DFMA warps/blk %2d x2 blk/SM: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  {
    int iters = 10000;
    barrier_loop<<<sms, 256>>>(10); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); barrier_loop<<<sms, 256>>>(iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("grid barrier (%d CTAs): %.3f us\n", sms, ms * 1000 / iters);
  }
  {
    size_t bytes = 800ull << 20; double2* x; CK(cudaMalloc(&x, bytes)); CK(cudaMemset(x, 0, bytes));
    for (int tpb : {256, 512, 1024}) for (int bps : {1, 2, 4}) {
      stream_read<<<sms * bps, tpb>>>(x, bytes / 16, out); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); for (int r = 0; r < 5; r++) stream_read<<<sms * bps, tpb>>>(x, bytes / 16, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("stream read 800MB tpb %d blk/SM %d: %.1f GB/s\n", tpb, bps, 5.0 * bytes / ms / 1e6);
    }
  }
  return 0;
}
