// FP64 pipe microbenchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync f64) throughput.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; i++) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int K>
__device__ __forceinline__ void mma_f64(double (&d)[4], const double* a, const double* b) {
  if constexpr (K == 4) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
  } else if constexpr (K == 8) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  } else {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
}

template <int K, int NACC>
__global__ void dmma_kernel(double* out, int iters) {
  double a[K / 2], b[K / 4];
#pragma unroll
  for (int i = 0; i < K / 2; i++) a[i] = 1.0 + 1e-12 * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < K / 4; i++) b[i] = 1e-12 * (threadIdx.x - i);
  double d[NACC][4];
#pragma unroll
  for (int j = 0; j < NACC; j++)
#pragma unroll
    for (int i = 0; i < 4; i++) d[j][i] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < NACC; j++) mma_f64<K>(d[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < NACC; j++)
#pragma unroll
    for (int i = 0; i < 4; i++) s += d[j][i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clockRate %d kHz\n", p.name, p.multiProcessorCount, clk);
  double* out; CK(cudaMalloc(&out, 4096 * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int rep = 0; rep < 2; rep++) {
    for (int bpsm : {1, 2, 4}) {
      for (int threads : {128, 256, 512}) {
        int iters = 20000;
        int grid = sms * bpsm;
        dfma_kernel<<<grid, threads>>>(out, 100, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        dfma_kernel<<<grid, threads>>>(out, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 16 * iters * (double)grid * threads;
        printf("DFMA grid=%d thr=%d : %.2f TFLOP/s (%.3f ms)\n", grid, threads, fl / ms / 1e9, ms);
      }
    }
  }
#define RUN_MMA(K, NACC)                                                                         \
  for (int bpsm : {1, 2, 4}) for (int threads : {128, 256}) {                                    \
      int iters = 4000; int grid = sms * bpsm;                                                   \
      dmma_kernel<K, NACC><<<grid, threads>>>(out, 10);                                          \
      cudaEventRecord(e0);                                                                       \
      dmma_kernel<K, NACC><<<grid, threads>>>(out, iters);                                       \
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));                                         \
      float ms; cudaEventElapsedTime(&ms, e0, e1);                                               \
      double fl = 2.0 * 16 * 8 * K * (double)NACC * iters * grid * (threads / 32);               \
      printf("DMMA m16n8k%d nacc=%d grid=%d thr=%d : %.2f TFLOP/s (%.3f ms)\n", K, NACC, grid,   \
             threads, fl / ms / 1e9, ms);                                                        \
    }
  RUN_MMA(4, 4) RUN_MMA(4, 8) RUN_MMA(8, 4) RUN_MMA(8, 8) RUN_MMA(16, 4) RUN_MMA(16, 8)
  // sustained: DMMA k8 for ~4 s
  {
    int grid = sms * 2, threads = 256, iters = 40000;
    float tot = 0; double fl = 0;
    for (int r = 0; r < 10; r++) {
      cudaEventRecord(e0);
      dmma_kernel<8, 8><<<grid, threads>>>(out, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      tot += ms; fl += 2.0 * 16 * 8 * 8 * 8.0 * iters * grid * (threads / 32);
      printf("sustained DMMA k8 rep %d: %.2f TFLOP/s (%.1f ms)\n", r, 2.0 * 16 * 8 * 8 * 8.0 * iters * grid * (threads / 32) / ms / 1e9, ms);
    }
    printf("sustained DMMA avg %.2f TFLOP/s over %.1f s\n", fl / tot / 1e9, tot / 1e3);
    tot = 0; fl = 0;
    for (int r = 0; r < 10; r++) {
      cudaEventRecord(e0);
      dfma_kernel<<<grid, threads>>>(out, 200000, 1.0000001, 1e-9);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      tot += ms; fl += 2.0 * 16 * 200000.0 * grid * threads;
    }
    printf("sustained DFMA avg %.2f TFLOP/s over %.1f s\n", fl / tot / 1e9, tot / 1e3);
  }
  return 0;
}
