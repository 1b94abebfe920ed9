// Scratch experiment (not product): is the SoA 19-plane access pattern
// itself below the flat-copy bandwidth?  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
constexpr int Q = 19;
struct P19 { const float* s[Q]; float* d[Q]; };
__global__ void flat(const float4* __restrict__ s, float4* __restrict__ d, long long n4) {
  const long long i0 = (long long)blockIdx.x * blockDim.x * 4 + threadIdx.x;
  float4 v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) { long long i = i0 + (long long)k * blockDim.x; if (i < n4) v[k] = __ldcs(s + i); }
#pragma unroll
  for (int k = 0; k < 4; ++k) { long long i = i0 + (long long)k * blockDim.x; if (i < n4) __stcs(d + i, v[k]); }
}
// one thread per node, 19 planes (the step kernel's memory pattern without compute)
template <int CS>
__global__ void __launch_bounds__(128, 12) planes(P19 p, unsigned nxp, unsigned ny) {
  const unsigned x = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned s = ((unsigned)blockIdx.z * ny + blockIdx.y) * nxp + x;
  float v[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) v[i] = CS ? __ldcs(p.s[i] + s) : __ldg(p.s[i] + s);
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i) acc += v[i];
#pragma unroll
  for (int i = 0; i < Q; ++i) { if (CS) __stcs(p.d[i] + s, v[i] + acc * 1e-30f); else p.d[i][s] = v[i] + acc * 1e-30f; }
}
// AoSoA: blocks of 32 nodes x 19 directions contiguous (2432 B per block)
__global__ void __launch_bounds__(128, 12) aosoa(const float* __restrict__ s, float* __restrict__ d, long long nblk) {
  const long long b = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= nblk) return;
  const float* sb = s + b * (Q * 32);
  float* db = d + b * (Q * 32);
  float v[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) v[i] = __ldg(sb + i * 32 + lane);
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i) acc += v[i];
#pragma unroll
  for (int i = 0; i < Q; ++i) db[i * 32 + lane] = v[i] + acc * 1e-30f;
}
int main() {
  const unsigned nx = 512, ny = 512, nz = 512;
  const long long N = (long long)nx * ny * nz, tot = N * Q;
  float *a, *b;
  cudaMalloc(&a, tot * 4); cudaMalloc(&b, tot * 4);
  cudaMemset(a, 0, tot * 4); cudaMemset(b, 0, tot * 4);
  P19 p;
  for (int i = 0; i < Q; ++i) { p.s[i] = a + i * N; p.d[i] = b + i * N; }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto time = [&](const char* name, auto launch) {
    for (int k = 0; k < 3; ++k) launch();
    cudaEventRecord(e0);
    const int R = 20;
    for (int k = 0; k < R; ++k) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %8.1f GB/s  (%.3f ms)\n", name, 2.0 * tot * 4 * R / (ms / 1e3) / 1e9, ms / R);
  };
  time("flat float4 one-pass", [&] { flat<<<(unsigned)((tot / 4 + 1023) / 1024), 256>>>((const float4*)a, (float4*)b, tot / 4); });
  time("19 planes, thread/node", [&] { planes<0><<<dim3(nx / 128, ny, nz), 128>>>(p, nx, ny); });
  time("19 planes, .cs hints", [&] { planes<1><<<dim3(nx / 128, ny, nz), 128>>>(p, nx, ny); });
  time("AoSoA 32-node blocks", [&] { aosoa<<<(unsigned)(N / 128), 128>>>(a, b, N / 32); });
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
