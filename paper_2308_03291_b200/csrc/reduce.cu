// Expected score of a distribution's marginals under a potential tensor,
// sum_e p(e) theta(e) per instance -- the reduction behind cross-entropy,
// entropy and KL (dist.py:306-347, _expected_score_under via masked_dot,
// numerics.py:171-183: parts with p(e) = 0 contribute 0 even where theta is
// -inf; a part with p(e) > 0 and theta = -inf makes the sum -inf, i.e. the
// cross-entropy +inf).  The marginals stay on the device: only B doubles and
// B flags come back.
#include "common.cuh"

namespace {

constexpr int kRT = 256;

template <typename T>  // float: the batched path; double: the exact mode
__global__ void __launch_bounds__(kRT) masked_dot_kernel(const T* __restrict__ marg, const T* __restrict__ theta,
                                                         int64_t len, double* __restrict__ out,
                                                         int32_t* __restrict__ neginf) {
  const int b = blockIdx.y;
  const T* p = marg + (size_t)b * len;
  const T* t = theta + (size_t)b * len;
  double acc = 0.0;
  int ninf_hit = 0;
  for (int64_t e = (int64_t)blockIdx.x * kRT + threadIdx.x; e < len; e += (int64_t)gridDim.x * kRT) {
    const T pe = __ldg(p + e);
    if (pe > (T)0) {
      const T te = __ldg(t + e);
      if ((double)te == ninfd()) ninf_hit = 1;
      else acc = fma((double)pe, (double)te, acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  ninf_hit = __any_sync(0xffffffffu, ninf_hit);
  __shared__ double red[kRT / 32];
  __shared__ int redf[kRT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    red[warp] = acc;
    redf[warp] = ninf_hit;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    int f = 0;
    for (int w = 0; w < kRT / 32; ++w) {
      s += red[w];
      f |= redf[w];
    }
    atomicAdd(out + b, s);
    if (f) atomicOr(neginf + b, 1);
  }
}

}  // namespace

// out[b] += sum_e marg[b][e] theta[b][e] over marg > 0; neginf[b] |= (a marked part is -inf).
// out / neginf are accumulated into (the caller zeroes them once for several tensors).
extern "C" int sdb_masked_dot(const float* marg, const float* theta, int64_t B, int64_t len, double* out,
                              int32_t* neginf, void* stream) {
  if (B < 0 || len < 0 || (B > 0 && len > 0 && (!marg || !theta || !out || !neginf))) return SDB_ERR_ARG;
  if (B == 0 || len == 0) return SDB_OK;
  const int64_t per = (len + kRT - 1) / kRT;
  const unsigned gx = (unsigned)(per < 64 ? per : 64);
  masked_dot_kernel<float><<<dim3(gx, (unsigned)B), kRT, 0, (cudaStream_t)stream>>>(marg, theta, len, out, neginf);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

// exact mode: float64 marginals and potentials
extern "C" int sdb_masked_dot_f64(const double* marg, const double* theta, int64_t B, int64_t len, double* out,
                                  int32_t* neginf, void* stream) {
  if (B < 0 || len < 0 || (B > 0 && len > 0 && (!marg || !theta || !out || !neginf))) return SDB_ERR_ARG;
  if (B == 0 || len == 0) return SDB_OK;
  const int64_t per = (len + kRT - 1) / kRT;
  const unsigned gx = (unsigned)(per < 64 ? per : 64);
  masked_dot_kernel<double><<<dim3(gx, (unsigned)B), kRT, 0, (cudaStream_t)stream>>>(marg, theta, len, out, neginf);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
