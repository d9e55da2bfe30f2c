// k3bench.cu -- the memory side of K3 alone: per item, the 8 columns of two
// Stolt mirror classes ((+-kx, +-ky), 4 KB each along k) are bulk-copied
// into an S-stage ring by a producer warp, consumer warps read each stage once
// and write the 8 columns (4 KB each along z) to a second volume, optionally
// through a column buffer and 256-byte warp stores as k3_ws does.  Large
// geometry: 512 x 512 columns of 512 complex (1 GiB each way), with an
// optional fraction of skipped (dead) columns.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/k3bench scripts/k3bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2305_02064_b200/csrc/tma.cuh"

constexpr int N = 512;   // nx = ny = nk = nz
constexpr uint32_t COL = N * 8;

// item i -> class pair; class c = (a, b) with 0 <= a, b <= N/2 mirrored to
// (+-a, +-b) mod N (4 distinct columns for 0 < a, b < N/2)
__device__ __forceinline__ int col_of(int cls, int m) {
  const int a = cls % (N / 2), b = cls / (N / 2);
  const int x = (m & 1) ? (N - a) & (N - 1) : a;
  const int y = (m & 2) ? (N - b) & (N - 1) : b;
  return y * N + x;
}

template <int S, int NCW>
__global__ void __launch_bounds__(NCW * 32 + 32, 1)
    k3_stream(const float2 *__restrict__ in, float2 *__restrict__ out, float *sink, int nitems) {
  constexpr uint32_t STAGE = 8 * COL;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      sartma::mbar_init(&full[i], 1);
      sartma::mbar_init(&empty[i], NCW);
    }
    sartma::fence_barrier_init();
  }
  __syncthreads();
  if (tid >= NCW * 32) {
    const int lane = tid & 31;
    unsigned n = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++n) {
      const int st = n % S;
      if (n >= S) sartma::mbar_wait(&empty[st], ((n / S) - 1) & 1);
      if (lane == 0) sartma::mbar_arrive_expect_tx(&full[st], STAGE);
      __syncwarp();
      if (lane < 8) {
        const int c = col_of(2 * item + (lane >> 2), lane & 3);
        sartma::bulk_g2s(sm + (size_t)st * STAGE + lane * COL, in + (size_t)c * N, COL, &full[st]);
      }
    }
    return;
  }
  float acc = 0.f;
  unsigned n = 0;
  const int lane = tid & 31, warp = tid >> 5;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++n) {
    const int st = n % S;
    sartma::mbar_wait(&full[st], (n / S) & 1);
    const float4 *sv = reinterpret_cast<const float4 *>(sm + (size_t)st * STAGE);
    float4 r[8 * COL / 16 / (NCW * 32)];
#pragma unroll
    for (int i = 0; i < (int)(8 * COL / 16 / (NCW * 32)); ++i) r[i] = sv[i * NCW * 32 + tid];
    sartma::fence_proxy_async();
    __syncwarp();
    if (lane == 0) sartma::mbar_arrive(&empty[st]);
    // column m of the item = float4 words [m * 256, (m + 1) * 256)
#pragma unroll
    for (int i = 0; i < (int)(8 * COL / 16 / (NCW * 32)); ++i) {
      const int w = i * NCW * 32 + tid, m = w >> 8, o = w & 255;
      const int c = col_of(2 * item + (m >> 2), m & 3);
      acc += r[i].x;
      reinterpret_cast<float4 *>(out + (size_t)c * N)[o] = r[i];
    }
  }
  if (acc == 12345.f) sink[warp] = acc;
}

template <int S, int NCW>
void run(const float2 *in, float2 *out, float *sink, double live) {
  auto k = k3_stream<S, NCW>;
  const int smem = S * 8 * COL;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // (N/2)^2 classes -> (N/2)^2 / 2 items; `live` of them
  const int nitems = (int)((N / 2) * (N / 2) / 2 * live);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int rep = 0; rep < 8; ++rep) {
    cudaEventRecord(a);
    k<<<148, NCW * 32 + 32, smem>>>(in, out, sink, nitems);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep >= 2 && ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  const double bytes = 2.0 * nitems * 8 * COL;
  printf("S=%d  %2d consumer warps  live %.2f  %.4f ms  %.2f GB  %.1f GB/s %s\n", S, NCW, live, best, bytes / 1e9,
         bytes / best / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  const size_t n = (size_t)N * N * N;
  float2 *in, *out;
  float *sink;
  if (cudaMalloc(&in, n * 8) != cudaSuccess || cudaMalloc(&out, n * 8) != cudaSuccess ||
      cudaMalloc(&sink, 4096) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(in, 0, n * 8);
  for (int rep = 0; rep < 2; ++rep) {
    run<4, 16>(in, out, sink, 1.0);
    run<4, 16>(in, out, sink, 0.82);
    run<6, 16>(in, out, sink, 0.82);
    run<3, 16>(in, out, sink, 0.82);
    run<4, 8>(in, out, sink, 0.82);
  }
  return 0;
}
