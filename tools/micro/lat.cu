// Microbenchmark: latency of the primitives the per-step DP loops are built
// from (one CTA, clock64 around N iterations).  Dev tool, not part of the build.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat lat.cu && ./lat
#include <cstdio>
#include <cuda_runtime.h>

template <int kMode>
__global__ void k(int iters, float* out, long long* cyc) {
  __shared__ float sm[1024];
  __shared__ double smd[64];
  const int t = threadIdx.x;
  for (int i = t; i < 1024; i += blockDim.x) sm[i] = 0.f;
  if (t < 64) smd[t] = 1.0;
  __syncthreads();
  float v = t * 1e-9f;
  double d = v;
  int idx = t & 31;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (kMode == 0) {          // bar.sync
      __syncthreads();
    } else if (kMode == 1) {   // dependent LDS chain (pointer chasing)
      idx = __float_as_int(sm[idx]) + (t & 31);
    } else if (kMode == 2) {   // dependent SHFL chain
      v = __shfl_xor_sync(0xffffffffu, v, 1) + 1.f;
    } else if (kMode == 3) {   // dependent FFMA chain
      v = fmaf(v, 1.0000001f, 1e-7f);
    } else if (kMode == 4) {   // dependent DADD chain
      d = d + 1e-9;
    } else if (kMode == 5) {   // STS then bar.sync then LDS (smem handoff through a barrier)
      sm[t] = v;
      __syncthreads();
      v = sm[(t + 1) & (blockDim.x - 1)] + 1.f;
    } else if (kMode == 6) {   // __syncwarp + smem handoff
      sm[t] = v;
      __syncwarp();
      v = sm[(t + 1) & 31 | (t & ~31)] + 1.f;
    } else if (kMode == 7) {   // DSETP + select chain (max-plus compare)
      const double c = smd[i & 63] + d;
      d = (c > d) ? c : d - 1.0;
    }
  }
  long long t1 = clock64();
  if (t == 0) cyc[0] = t1 - t0;
  out[t] = v + (float)d + idx;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4096 * 4);
  cudaMallocManaged(&cyc, 8);
  const char* names[] = {"bar.sync", "LDS chain", "SHFL chain", "FFMA chain", "DADD chain", "STS+bar+LDS",
                         "STS+syncwarp+LDS", "LDS.64+DADD+DSETP chain"};
  for (int threads : {32, 64, 256, 512}) {
    for (int mode = 0; mode < 8; ++mode) {
      const int iters = 4096;
      void (*f)(int, float*, long long*) = nullptr;
      switch (mode) {
        case 0: f = k<0>; break; case 1: f = k<1>; break; case 2: f = k<2>; break; case 3: f = k<3>; break;
        case 4: f = k<4>; break; case 5: f = k<5>; break; case 6: f = k<6>; break; default: f = k<7>; break;
      }
      f<<<1, threads>>>(iters, out, cyc);
      f<<<1, threads>>>(iters, out, cyc);
      cudaDeviceSynchronize();
      printf("threads=%3d %-26s %.1f cycles/iter\n", threads, names[mode], (double)cyc[0] / iters);
    }
  }
  return 0;
}
