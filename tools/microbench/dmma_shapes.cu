// Microbenchmark: FP64 mma.sync shapes on sm_100a (m8n8k4 vs m16n8k4 / k8 / k16): FLOP/s with
// register operands, 8 independent accumulators per warp.  Decides the ADMM kernel's MMA shape.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

template <int SHAPE>
__global__ void loop(double* out, int iters, int skip_smsp = -1) {
  if (skip_smsp >= 0 && (threadIdx.x >> 5) % 4 == skip_smsp) return;
  double a[8], b[4], c[8][4];
  for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; i++) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) c[i][j] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (SHAPE == 0)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a[0]), "d"(b[0]));
      else if (SHAPE == 1)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      else if (SHAPE == 2)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0; for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) s += c[i][j];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d; CK(cudaMalloc(&d, 8));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const char* names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  const double flops_per[4] = {2.0*8*8*4, 2.0*16*8*4, 2.0*16*8*8, 2.0*16*8*16};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    for (int sh = 0; sh < 4; sh++) {
      const int iters = 4000;
      auto launch = [&]() {
        if (sh == 0) loop<0><<<sms, 32 * warps>>>(d, iters);
        else if (sh == 1) loop<1><<<sms, 32 * warps>>>(d, iters);
        else if (sh == 2) loop<2><<<sms, 32 * warps>>>(d, iters);
        else loop<3><<<sms, 32 * warps>>>(d, iters);
      };
      launch(); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = flops_per[sh] * 8.0 * iters * warps * sms;
      printf("%-9s warps/SM %2d: %.2f TFLOP/s\n", names[sh], warps, fl / (ms * 1e-3) / 1e12);
    }
  }
  // DMMA issue from 3 of the 4 SM sub-partitions (warp w runs on SMSP w % 4): is the FP64 tensor
  // throughput per sub-partition?
  for (int warps : {8, 16}) {
    const int iters = 4000;
    for (int skip : {-1, 3}) {
      loop<0><<<sms, 32 * warps>>>(d, iters, skip); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); loop<0><<<sms, 32 * warps>>>(d, iters, skip); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const int active = skip < 0 ? warps : warps - warps / 4;
      double fl = flops_per[0] * 8.0 * iters * active * sms;
      printf("m8n8k4 warps/SM %2d skip SMSP %2d: %.2f TFLOP/s\n", warps, skip, fl / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
