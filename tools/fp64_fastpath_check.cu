// fp64_fastpath_check.cu -- checks the branch-free fast paths of the fp64
// division and square root (csrc/dual_kernels.cuh ddiv_fast / dsqrt_fast)
// against the IEEE operations (x / d, sqrt(x)) on the B200: wherever the fast
// path reports ok, its result must be bitwise the IEEE result.  Operands:
// random 64-bit patterns (every exponent, both signs, specials), and the
// ranges the adaptive optimisers produce (numerators ~ |alpha m|, 1e-30..1e3;
// divisors sqrt(v) + eps with eps = 1e-8).  Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -I../paper_2406_13191_b200/csrc \
//        fp64_fastpath_check.cu -o fp64_fastpath_check && ./fp64_fastpath_check [rounds]
#include <cstdio>
#include <cstdlib>

#include "dual_kernels.cuh"

using namespace dcopf;

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {  // splitmix64
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double operand(unsigned long long r, int kind) {
  if (kind == 0) return __longlong_as_double((long long)r);  // any bit pattern
  // a log-uniform magnitude in [2^lo, 2^hi), random sign for kind 1
  const int lo = kind == 1 ? -100 : -27, hi = kind == 1 ? 12 : 10;
  const double u = (double)(r >> 11) * 0x1p-53;
  const double m = exp2(lo + (hi - lo) * u);
  return (kind == 1 && (r & 1)) ? -m : m;
}

// the fast paths and the IEEE operations in separate kernels (in one kernel
// ptxas merges the identical instruction sequences, which would compare a
// register with itself)
__device__ __forceinline__ void operands(unsigned long long seed, long i, double &x, double &d, double &s) {
  const unsigned long long r1 = mix(seed ^ (2 * i)), r2 = mix(seed ^ (2 * i + 1));
  const int kind = (int)(i % 3);
  x = operand(r1, kind);
  // divisor: random pattern (kind 0) or sqrt(v) + 1e-8 over the optimiser's range
  d = kind == 0 ? operand(r2, 0) : sqrt(operand(r2, 2)) + 1e-8;
  s = kind == 0 ? x : fabs(x);
}
__global__ void k_fast(unsigned long long seed, long n, double *q, double *r, unsigned char *ok) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    double x, d, s;
    operands(seed, i, x, d, s);
    bool o1 = true, o2 = true;
    q[i] = ddiv_fast(x, d, o1);
    r[i] = dsqrt_fast(s, o2);
    ok[i] = (unsigned char)(o1 | (o2 << 1));
  }
}
__global__ void k_ieee(unsigned long long seed, long n, double *q, double *r) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    double x, d, s;
    operands(seed, i, x, d, s);
    q[i] = x / d;
    r[i] = sqrt(s);
  }
}
__global__ void k_cmp(long n, const double *qf, const double *rf, const unsigned char *ok, const double *qi,
                      const double *ri, unsigned long long *cnt) {
  // cnt: [0] div fast, [1] div mismatches, [2] div slow, [3] sqrt fast, [4] sqrt mismatches, [5] sqrt slow
  unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    if (ok[i] & 1) {
      ++c[0];
      c[1] += __double_as_longlong(qf[i]) != __double_as_longlong(qi[i]);
    } else {
      ++c[2];
    }
    if (ok[i] & 2) {
      ++c[3];
      c[4] += __double_as_longlong(rf[i]) != __double_as_longlong(ri[i]);
    } else {
      ++c[5];
    }
  }
  for (int j = 0; j < 6; ++j) atomicAdd(&cnt[j], c[j]);
}

int main(int argc, char **argv) {
  const int rounds = argc > 1 ? atoi(argv[1]) : 64;
  const long n = 1L << 25;
  unsigned long long *d_cnt, h[6] = {0, 0, 0, 0, 0, 0};
  double *qf, *rf, *qi, *ri;
  unsigned char *ok;
  cudaMalloc(&d_cnt, sizeof h);
  cudaMalloc(&qf, n * 8);
  cudaMalloc(&rf, n * 8);
  cudaMalloc(&qi, n * 8);
  cudaMalloc(&ri, n * 8);
  cudaMalloc(&ok, n);
  cudaMemset(d_cnt, 0, sizeof h);
  for (int r = 0; r < rounds; ++r) {
    const unsigned long long seed = 0x5eedull * (r + 1);
    k_fast<<<148 * 8, 256>>>(seed, n, qf, rf, ok);
    k_ieee<<<148 * 8, 256>>>(seed, n, qi, ri);
    k_cmp<<<148 * 8, 256>>>(n, qf, rf, ok, qi, ri, d_cnt);
  }
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d_cnt, sizeof h, cudaMemcpyDeviceToHost);
  printf("{\"operands\": %ld, \"div_fast\": %llu, \"div_mismatch\": %llu, \"div_slow\": %llu, "
         "\"sqrt_fast\": %llu, \"sqrt_mismatch\": %llu, \"sqrt_slow\": %llu, \"cuda\": \"%s\"}\n",
         n * rounds, h[0], h[1], h[2], h[3], h[4], h[5], cudaGetErrorString(e));
  return (e == cudaSuccess && h[1] == 0 && h[4] == 0) ? 0 : 1;
}
