// fp64 throughput probe for the dense PTDF path: DFMA,
// DMMA m8n8k4 and m16n8k{4,8,16} issue rates on one B200.  Measurement only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void k_dfma(double *out, double s) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], s, 1e-7);
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r += a[i];
  if (r == 12345.0) out[0] = r;
}

__global__ void k_m8n8k4(double *out, double s) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0;
  double a = threadIdx.x * 1e-3, b = s;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += acc[i][0] + acc[i][1];
  if (r == 12345.0) out[0] = r;
}

__global__ void k_m16n8k4(double *out, double s) {
  double acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0;
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = s;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a0), "d"(a1), "d"(b));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (r == 12345.0) out[0] = r;
}

__global__ void k_m16n8k8(double *out, double s) {
  double acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0;
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = s, b1 = s + 1;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (r == 12345.0) out[0] = r;
}

template <class F>
static void run(const char *name, F kern, double flops_per_thread, int blocks, int threads) {
  double *out;
  cudaMalloc(&out, 8);
  kern<<<blocks, threads>>>(out, 0.999);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(out, 0.999);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 5.0 * flops_per_thread * blocks * threads;
  printf("%-10s blocks=%d threads=%d  %.2f TFLOP/s  (%s)\n", name, blocks, threads, fl / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int occ : {1, 2, 4}) {
    int blocks = sms * occ;
    run("dfma", k_dfma, 2.0 * 16 * kIters, blocks, 256);
    // per warp: 8 mma x 8*8*4 FMA x 2 flops per iteration; per thread /32
    run("m8n8k4", k_m8n8k4, 8.0 * 8 * 8 * 4 * 2 * kIters / 32, blocks, 256);
    run("m16n8k4", k_m16n8k4, 8.0 * 16 * 8 * 4 * 2 * kIters / 32, blocks, 256);
    run("m16n8k8", k_m16n8k8, 8.0 * 16 * 8 * 8 * 2 * kIters / 32, blocks, 256);
  }
  return 0;
}
