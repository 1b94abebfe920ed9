// Scratch experiment (not product): pull-pattern bandwidth, SoA planes vs
// AoSoA 32-node blocks (19 directions x 32 nodes contiguous), no collision.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int Q = 19;
__host__ __device__ constexpr int cx(int i) {
  return (i == 1 || i == 5 || i == 8 || i == 11 || i == 14) ? 1 : (i == 3 || i == 6 || i == 7 || i == 12 || i == 13) ? -1 : 0;
}
__host__ __device__ constexpr int cy(int i) {
  return (i == 2 || i == 5 || i == 6 || i == 15 || i == 18) ? 1 : (i == 4 || i == 7 || i == 8 || i == 16 || i == 17) ? -1 : 0;
}
__host__ __device__ constexpr int cz(int i) {
  return (i == 9 || i == 11 || i == 13 || i == 15 || i == 17) ? 1 : (i == 10 || i == 12 || i == 14 || i == 16 || i == 18) ? -1 : 0;
}
struct P19 { const float* s[Q]; float* d[Q]; };
// SoA: slot = ((z+1)*ny + y)*nx + x (ghost planes), interior y (1..ny-2), x wraps inside the row
template <int AOS>
__global__ void __launch_bounds__(128, 12) pull(P19 p, unsigned nx, unsigned ny, unsigned nz) {
  const unsigned x = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned y = blockIdx.y, z = blockIdx.z;
  const unsigned lane = threadIdx.x & 31;
  const unsigned s = ((z + 1) * ny + y) * nx + x;
  unsigned xm, xp, ym, yp, zm, zp, own;
  if (!AOS) {
    own = s;
    xm = x == 0 ? nx - 1 : (unsigned)-1;
    xp = x == nx - 1 ? (unsigned)-(int)(nx - 1) : 1u;
    ym = y == 0 ? 0u : (unsigned)-(int)nx;
    yp = y == ny - 1 ? 0u : nx;
    zm = (unsigned)-(int)(nx * ny);
    zp = nx * ny;
  } else {
    const unsigned B = Q * 32;  // elements per block
    own = (s >> 5) * B + (s & 31);
    xm = lane == 0 ? (x == 0 ? (nx / 32 - 1) * B + 31 : (unsigned)-(int)B + 31u) : (unsigned)-1;
    xp = lane == 31 ? (x == nx - 1 ? (unsigned)-(int)((nx / 32 - 1) * B + 31) : B - 31u) : 1u;
    ym = y == 0 ? 0u : (unsigned)-(int)(nx / 32 * B);
    yp = y == ny - 1 ? 0u : nx / 32 * B;
    zm = (unsigned)-(int)(nx * ny / 32 * B);
    zp = nx * ny / 32 * B;
  }
  float v[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const unsigned o = own + (cx(i) == 1 ? xm : cx(i) == -1 ? xp : 0u) + (cy(i) == 1 ? ym : cy(i) == -1 ? yp : 0u) +
                       (cz(i) == 1 ? zm : cz(i) == -1 ? zp : 0u);
    v[i] = __ldg(p.s[i] + o);
  }
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i) acc += v[i];
#pragma unroll
  for (int i = 0; i < Q; ++i) p.d[i][own] = v[i] + acc * 1e-30f;
}
int main() {
  const unsigned nx = 512, ny = 512, nz = 512;
  const long long S = (long long)nx * ny * (nz + 2), tot = S * Q;
  float *a, *b;
  cudaMalloc(&a, tot * 4); cudaMalloc(&b, tot * 4);
  cudaMemset(a, 0, tot * 4); cudaMemset(b, 0, tot * 4);
  P19 soa, aos;
  for (int i = 0; i < Q; ++i) { soa.s[i] = a + i * S; soa.d[i] = b + i * S; aos.s[i] = a + i * 32; aos.d[i] = b + i * 32; }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto time = [&](const char* name, auto launch) {
    for (int k = 0; k < 3; ++k) launch();
    cudaEventRecord(e0);
    const int R = 30;
    for (int k = 0; k < R; ++k) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = 2.0 * 19 * 4 * (double)nx * ny * nz;
    printf("%-28s %8.1f GB/s  (%.3f ms)\n", name, bytes * R / (ms / 1e3) / 1e9, ms / R);
  };
  for (int rep = 0; rep < 2; ++rep) {
    time("pull SoA planes", [&] { pull<0><<<dim3(nx / 128, ny, nz), 128>>>(soa, nx, ny, nz); });
    time("pull AoSoA 32-blocks", [&] { pull<1><<<dim3(nx / 128, ny, nz), 128>>>(aos, nx, ny, nz); });
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
