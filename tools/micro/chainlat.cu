// Microbenchmark: per-step latency of the alignment recurrence chain
// (SHFL + log-sum-exp of three terms) for one warp, with optional
// cp.async prefetch + wait_group per step.  Dev tool, not part of the build.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float lg2(float x) { float y; asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

template <int kMode, int kI = 1, bool kV16 = false, bool kBlkWait = false>
__global__ void k(const float* __restrict__ th, int steps, float* out, long long* cyc) {
  __shared__ __align__(16) float ring[kI][48 * 100];
  const int l = threadIdx.x & 31;
  float v[kI], o[kI], av[kI], lp[kI], lpo[kI];
  for (int q = 0; q < kI; ++q) v[q] = o[q] = av[q] = lp[q] = lpo[q] = 0.f;
  long long t0 = clock64();
  for (int s = 0; s < steps; s += 8) {
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
      for (int q = 0; q < kI; ++q) {
      if (kMode >= 1 && kV16) {
        const float* src = th + ((size_t)(s + kk) * 132 + q * 7 * 4) * 3 + 4 * l;
        uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring[q] + ((s + kk) % 48) * 100 + 4 * l);
        if (l < 25) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
      } else if (kMode >= 1) {
        const float* src = th + ((size_t)(s + kk) * 129 + l + q * 7) * 3;
        uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring[q] + ((s + kk) % 48) * 96 + l);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst + 128), "l"(src + 1));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst + 256), "l"(src + 2));
      }
      }
      if (kMode >= 1) {
        asm volatile("cp.async.commit_group;\n" ::);
        if (!kBlkWait) asm volatile("cp.async.wait_group 8;\n" ::);
        else if (kk == 0) asm volatile("cp.async.wait_group 8;\n" ::);
      }
#pragma unroll
      for (int q = 0; q < kI; ++q) {
      float x0 = 0.3f, x1 = -0.2f, x2 = 0.1f;
      if (kMode >= 1 && kV16) {
        const float* slot = ring[q] + ((s + kk + 40) % 48) * 100 + 3 * l;
        x0 = slot[0]; x1 = slot[1]; x2 = slot[2];
      } else if (kMode >= 1) {
        const float* slot = ring[q] + ((s + kk + 40) % 48) * 96 + l;
        x0 = slot[0]; x1 = slot[32]; x2 = slot[64];
      }
      float lv = __shfl_up_sync(0xffffffffu, v[q], 1);
      float lo = __shfl_up_sync(0xffffffffu, o[q], 1);
      float t0 = fmaf(x0, 1.44269504f, lp[q] + (lpo[q] - o[q]));
      float t1 = fmaf(x1, 1.44269504f, av[q]);
      float t2 = fmaf(x2, 1.44269504f, lv + (lo - o[q]));
      lp[q] = lv; lpo[q] = lo;
      float M = fmaxf(fmaxf(t0, t1), t2);
      float Mc = fmaxf(M, -1e30f);
      float r = M > -1e30f ? rintf(M) : 0.f;
      float e = ex2(t0 - Mc) + ex2(t1 - Mc) + ex2(t2 - Mc);
      v[q] = (Mc - r) + lg2(e);
      o[q] += r;
      av[q] = v[q];
      }
    }
    if (kMode >= 2) __syncthreads();
  }
  long long t1 = clock64();
  out[threadIdx.x] = v[0] + o[0] + (kI > 1 ? v[kI - 1] : 0.f);
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  const int steps = 4096;
  float *th, *out; long long* cyc;
  cudaMalloc(&th, (size_t)(steps + 64) * 132 * 3 * 4);
  cudaMemset(th, 0, (size_t)(steps + 64) * 132 * 3 * 4);
  cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8);
  long long h;
  const char* names[] = {"chain only", "chain + cp.async/wait per step", "chain + cp.async + barrier/8 (1 warp)", "same, 5 warps",
                         "ILP2 chain only", "ILP2 + cp.async (1 warp)", "ILP2 + cp.async + barrier, 5 warps", "ILP3 chain only", "ILP4 chain only", "v16: chain + cp.async (1 warp)", "v16: 5 warps + barrier", "v16: ILP2 1 warp", "v16: ILP2 5 warps + barrier", "v16 blkwait 1 warp", "v16 blkwait 5 warps", "v16 blkwait ILP2 5 warps", "v16 blkwait ILP2 1 warp"};
  for (int mode = 0; mode < 17; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      int thr = mode == 3 ? 160 : 32;
      if (mode == 0) k<0><<<1, thr>>>(th, steps, out, cyc);
      if (mode == 1) k<1><<<1, thr>>>(th, steps, out, cyc);
      if (mode == 2 || mode == 3) k<2><<<1, thr>>>(th, steps, out, cyc);
      if (mode == 4) k<0, 2><<<1, 32>>>(th, steps, out, cyc);
      if (mode == 5) k<1, 2><<<1, 32>>>(th, steps, out, cyc);
      if (mode == 6) k<2, 2><<<1, 160>>>(th, steps, out, cyc);
      if (mode == 7) k<0, 3><<<1, 32>>>(th, steps, out, cyc);
      if (mode == 8) k<0, 4><<<1, 32>>>(th, steps, out, cyc);
      if (mode == 9) k<1, 1, true><<<1, 32>>>(th, steps, out, cyc);
      if (mode == 10) k<2, 1, true><<<1, 160>>>(th, steps, out, cyc);
      if (mode == 11) k<1, 2, true><<<1, 32>>>(th, steps, out, cyc);
      if (mode == 12) k<2, 2, true><<<1, 160>>>(th, steps, out, cyc);
      if (mode == 13) k<1, 1, true, true><<<1, 32>>>(th, steps, out, cyc);
      if (mode == 14) k<2, 1, true, true><<<1, 160>>>(th, steps, out, cyc);
      if (mode == 15) k<2, 2, true, true><<<1, 160>>>(th, steps, out, cyc);
      if (mode == 16) k<1, 2, true, true><<<1, 32>>>(th, steps, out, cyc);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %.1f cycles/step\n", names[mode], (double)h / steps);
  }
  return 0;
}
