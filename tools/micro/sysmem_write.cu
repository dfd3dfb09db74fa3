// Dev micro-test: store patterns into pinned (mapped) host memory.
#include <cstdio>
#include <cuda_runtime.h>
// (a) warp writes 32 consecutive floats per instruction
__global__ void wa(float* p, size_t nf) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i < nf; i += (size_t)gridDim.x * blockDim.x) p[i] = 1.f;
}
// (b) half-warp rows of 48 floats written as 3 stride-12-byte instructions (lane q: floats 3q, 3q+1, 3q+2)
__global__ void wb(float* p, size_t nrows) {
  const int lane = threadIdx.x & 31, g = lane >> 4, q = lane & 15;
  size_t row = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) / 16;
  for (; row < nrows; row += (size_t)gridDim.x * blockDim.x / 16) {
    float* d = p + row * 48 + 3 * q;
    d[0] = 1.f; d[1] = 2.f; d[2] = 3.f;
  }
  (void)g;
}
// (c) same rows, lane q writes floats q, q+16, q+32 (64 contiguous bytes per instruction per half-warp)
__global__ void wc(float* p, size_t nrows) {
  const int q = threadIdx.x & 15;
  size_t row = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) / 16;
  for (; row < nrows; row += (size_t)gridDim.x * blockDim.x / 16) {
    float* d = p + row * 48;
    d[q] = 1.f; d[q + 16] = 2.f; d[q + 32] = 3.f;
  }
}
int main() {
  const size_t bytes = 203295744, nf = bytes / 4, nrows = nf / 48;
  float* h;
  cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int k = 0; k < 3; ++k) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (k == 0) wa<<<592, 256>>>(h, nf);
      if (k == 1) wb<<<592, 256>>>(h, nrows);
      if (k == 2) wc<<<592, 256>>>(h, nrows);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("pattern %c: %.3f ms  %.1f GB/s  (%s)\n", 'a' + k, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
