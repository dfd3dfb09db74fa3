// Dev micro-test: tcgen05.mma kind::tf32 with SWIZZLE_NONE K-major smem
// descriptors, D[128 x 32] in TMEM, 1xTF32 and 3xTF32 (hi/lo split) against
// an fp64 host reference.  Validates the descriptor conventions the PCFG
// contraction uses.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 umma_tf32.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: core matrix = 8 rows x 16 B contiguous; LBO = bytes between the
// two K-adjacent core matrices of one K=8 step, SBO = bytes between 8-row groups
__device__ __forceinline__ uint64_t kdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

template <int K>
__global__ void umma_test(const float* A, const float* B, float* D, int split) {
  extern __shared__ __align__(1024) uint8_t sm[];
  float* sAh = (float*)sm;
  float* sAl = sAh + 128 * K;
  float* sBh = sAl + 128 * K;
  float* sBl = sBh + 32 * K;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x;
  auto off = [](int r, int c) { return ((r / 8) * (K / 4) + c / 4) * 32 + (r % 8) * 4 + c % 4; };
  for (int e = tid; e < 128 * K; e += blockDim.x) {
    const int r = e / K, c = e % K;
    const float x = A[e], h = split ? tf32_rna(x) : x;
    sAh[off(r, c)] = h;
    sAl[off(r, c)] = x - h;
  }
  for (int e = tid; e < 32 * K; e += blockDim.x) {
    const int r = e / K, c = e % K;
    const float x = B[e], h = split ? tf32_rna(x) : x;
    sBh[off(r, c)] = h;
    sBl[off(r, c)] = x - h;
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t sbo = (K / 4) * 128;
    const int passes = split ? 3 : 1;
    int first = 1;
    for (int p = 0; p < passes; ++p) {
      const uint32_t a0 = su32(p == 2 ? sAl : sAh), b0 = su32(p == 1 ? sBl : sBh);
      for (int s = 0; s < K / 8; ++s) {
        const uint64_t ad = kdesc(a0 + s * 256, 128, sbo), bd = kdesc(b0 + s * 256, 128, sbo);
        const uint32_t acc = first ? 0u : 1u;
        first = 0;
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc_tf32(128, 32)), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar)));
  }
  {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(su32(&mbar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int w = tid >> 5, l = tid & 31;
  if (w < 4) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tmem + ((uint32_t)(32 * w) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 32; ++j) D[(32 * w + l) * 32 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  constexpr int K = 64;
  std::vector<float> A(128 * K), B(32 * K), D(128 * 32);
  srand(1);
  for (auto& x : A) x = (float)rand() / RAND_MAX * 2.f - 0.5f;
  for (auto& x : B) x = (float)rand() / RAND_MAX * 1.5f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const size_t smem = (size_t)(2 * 128 * K + 2 * 32 * K) * 4;
  cudaFuncSetAttribute(umma_test<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int split = 0; split < 2; ++split) {
    cudaMemset(dD, 0, D.size() * 4);
    umma_test<K><<<1, 128, smem>>>(dA, dB, dD, split);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxrel = 0, maxabs = 0;
    for (int i = 0; i < 128; ++i)
      for (int j = 0; j < 32; ++j) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)A[i * K + k] * (double)B[j * K + k];
        const double err = fabs(D[i * 32 + j] - ref);
        maxabs = fmax(maxabs, err);
        maxrel = fmax(maxrel, err / fmax(fabs(ref), 1e-3));
      }
    printf("split=%d max_abs=%.3e max_rel=%.3e  D[0]=%f D[last]=%f\n", split, maxabs, maxrel, D[0], D[128 * 32 - 1]);
  }
  return 0;
}
