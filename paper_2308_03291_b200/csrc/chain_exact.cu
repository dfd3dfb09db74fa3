// Exact mode (float64 in, float64 out) for the linear-chain and semi-Markov
// CRFs: the reference recurrences restated one-for-one in fp64, one CTA per
// instance, a thread per tag, the lattices in the workspace.  This is the
// drop-in for callers that hand the reference float64 potentials and compare
// at its own tolerances (1e-9); the batched fp32 kernels (chain.cu,
// semimarkov.cu) remain the throughput path.
//
//   chain  (structdist chain.py:64-95): alpha_(t+1)[b] = lse_a alpha_t[a] + theta_t[a,b],
//          beta_t[a] = lse_b theta_t[a,b] + beta_(t+1)[b], p = exp(alpha + theta + beta - Z);
//   semi-Markov (chain.py:250-298): alpha[t,l] = lse_{w<=min(s,t),p} alpha[t-w,p] +
//          theta[t-w,w-1,p,l] with the virtual start alpha[0,0] = 0; beta over the
//          segments that start at t; p = exp(alpha[t,p] + theta + beta[t+w,l] - Z).
#include "common.cuh"

namespace {

constexpr int kT = 256;

struct LseD {  // max-shifted log-sum-exp of a stream of fp64 terms (-inf-safe)
  double mx = ninfd(), s = 0.0;
  __device__ void add(double x) {
    if (x == ninfd()) return;
    if (x > mx) { s = s * exp(mx - x) + 1.0; mx = x; } else { s += exp(x - mx); }
  }
  __device__ double get() const { return mx == ninfd() ? ninfd() : mx + log(s); }
};

__device__ double block_lse(double v, double* red) {  // every thread's v -> lse over the block
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double mx = v;
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  double M = ninfd();
  for (int w = 0; w < nw; ++w) M = fmax(M, red[w]);
  __syncthreads();
  double s = (v == ninfd() || M == ninfd()) ? 0.0 : exp(v - M);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  double S = 0.0;
  for (int w = 0; w < nw; ++w) S += red[w];
  __syncthreads();
  return M == ninfd() ? ninfd() : M + log(S);
}

__global__ void __launch_bounds__(kT) chain_exact_kernel(const double* __restrict__ init_all,
                                                         const double* __restrict__ trans_all, int n, int m,
                                                         double* __restrict__ ws, double* __restrict__ logz,
                                                         double* __restrict__ minit_all,
                                                         double* __restrict__ mtrans_all, int32_t* __restrict__ status) {
  __shared__ double red[kT / 32];
  __shared__ int bad_s;
  const int b = blockIdx.x, tid = threadIdx.x;
  const size_t mm = (size_t)m * m;
  const double* init = init_all + (size_t)b * m;
  const double* tr = trans_all + (size_t)b * (n - 1) * mm;
  double* al = ws + (size_t)b * 2 * n * m;
  double* be = al + (size_t)n * m;
  if (tid == 0) bad_s = 0;
  __syncthreads();
  {
    int bad = 0;
    for (int e = tid; e < m; e += kT) bad |= bad_value(init[e]);
    for (size_t e = tid; e < (size_t)(n - 1) * mm; e += kT) bad |= bad_value(tr[e]);
    if (bad) bad_s = 1;
  }
  for (int a = tid; a < m; a += kT) al[a] = init[a];
  __syncthreads();
  for (int t = 0; t + 1 < n; ++t) {  // chain.py:64-70
    const double* th = tr + (size_t)t * mm;
    for (int c = tid; c < m; c += kT) {
      LseD acc;
      for (int a = 0; a < m; ++a) acc.add(al[(size_t)t * m + a] + th[(size_t)a * m + c]);
      al[(size_t)(t + 1) * m + c] = acc.get();
    }
    __syncthreads();
  }
  double part = ninfd();
  {
    LseD acc;
    for (int c = tid; c < m; c += kT) acc.add(al[(size_t)(n - 1) * m + c]);
    part = acc.get();
  }
  const double z = block_lse(part, red);
  const bool bad = bad_s != 0;
  if (tid == 0) {
    logz[b] = z;
    status[b] = bad ? SDB_ST_INVALID : (z == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
  }
  if (!minit_all) return;
  double* pi = minit_all + (size_t)b * m;
  double* pt = mtrans_all ? mtrans_all + (size_t)b * (n - 1) * mm : nullptr;
  const bool zok = !bad && z != ninfd();
  for (int a = tid; a < m; a += kT) be[(size_t)(n - 1) * m + a] = 0.0;
  __syncthreads();
  for (int t = n - 2; t >= 0; --t) {  // chain.py:73-77
    const double* th = tr + (size_t)t * mm;
    for (int a = tid; a < m; a += kT) {
      LseD acc;
      for (int c = 0; c < m; ++c) acc.add(th[(size_t)a * m + c] + be[(size_t)(t + 1) * m + c]);
      be[(size_t)t * m + a] = acc.get();
    }
    __syncthreads();
  }
  for (int a = tid; a < m; a += kT) pi[a] = zok ? exp(init[a] + be[a] - z) : 0.0;  // chain.py:91-94
  if (pt)
    for (size_t e = tid; e < (size_t)(n - 1) * mm; e += kT) {
      const size_t t = e / mm, r = e - t * mm, a = r / m, c = r - a * m;
      pt[e] = zok ? exp(al[t * m + a] + tr[e] + be[(t + 1) * m + c] - z) : 0.0;
    }
}

__global__ void __launch_bounds__(kT) semimarkov_exact_kernel(const double* __restrict__ th_all, int n, int s, int m,
                                                              double* __restrict__ ws, double* __restrict__ logz,
                                                              double* __restrict__ marg_all,
                                                              int32_t* __restrict__ status) {
  __shared__ double red[kT / 32];
  __shared__ int bad_s;
  const int b = blockIdx.x, tid = threadIdx.x;
  const size_t mm = (size_t)m * m, seg = (size_t)s * mm;  // theta [n][s][m prev][m label]
  const double* th = th_all + (size_t)b * n * seg;
  double* al = ws + (size_t)b * 2 * (n + 1) * m;
  double* be = al + (size_t)(n + 1) * m;
  if (tid == 0) bad_s = 0;
  __syncthreads();
  {
    int bad = 0;
    for (size_t e = tid; e < (size_t)n * seg; e += kT) bad |= bad_value(th[e]);
    if (bad) bad_s = 1;
  }
  for (int l = tid; l < m; l += kT) al[l] = (l == 0) ? 0.0 : ninfd();  // virtual start (chain.py:256-258)
  __syncthreads();
  for (int t = 1; t <= n; ++t) {  // chain.py:259-265
    for (int l = tid; l < m; l += kT) {
      LseD acc;
      for (int w = 1; w <= min(s, t); ++w) {
        const double* a = al + (size_t)(t - w) * m;
        const double* x = th + (size_t)(t - w) * seg + (size_t)(w - 1) * mm + l;
        for (int p = 0; p < m; ++p) acc.add(a[p] + x[(size_t)p * m]);
      }
      al[(size_t)t * m + l] = acc.get();
    }
    __syncthreads();
  }
  double part;
  {
    LseD acc;
    for (int l = tid; l < m; l += kT) acc.add(al[(size_t)n * m + l]);
    part = acc.get();
  }
  const double z = block_lse(part, red);
  const bool bad = bad_s != 0;
  if (tid == 0) {
    logz[b] = z;
    status[b] = bad ? SDB_ST_INVALID : (z == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
  }
  if (!marg_all) return;
  double* mg = marg_all + (size_t)b * n * seg;
  const bool zok = !bad && z != ninfd();
  for (int l = tid; l < m; l += kT) be[(size_t)n * m + l] = 0.0;
  __syncthreads();
  for (int t = n - 1; t >= 0; --t) {  // chain.py:272-282
    for (int p = tid; p < m; p += kT) {
      LseD acc;
      for (int w = 1; w <= min(s, n - t); ++w) {
        const double* x = th + (size_t)t * seg + (size_t)(w - 1) * mm + (size_t)p * m;
        const double* bb = be + (size_t)(t + w) * m;
        for (int l = 0; l < m; ++l) acc.add(x[l] + bb[l]);
      }
      be[(size_t)t * m + p] = acc.get();
    }
    __syncthreads();
  }
  for (size_t e = tid; e < (size_t)n * seg; e += kT) {  // chain.py:285-298
    const size_t t = e / seg, r = e - t * seg, w = r / mm, r2 = r - w * mm, p = r2 / m, l = r2 - p * m;
    double v = 0.0;
    if (zok && (int)(t + w + 1) <= n) v = exp(al[t * m + p] + th[e] + be[(t + w + 1) * m + l] - z);
    mg[e] = v;
  }
}

}  // namespace

extern "C" size_t sdb_chain_fb_f64_workspace(int64_t B, int32_t n, int32_t m) {
  return (B < 0 || n < 1 || m < 1) ? 0 : (size_t)B * 2 * n * m * sizeof(double) + 256;
}
// chain.py:64-95 in fp64: init [B,m], trans [B,n-1,m,m] float64; marg_init / marg_trans nullable
extern "C" int sdb_chain_fb_f64(const double* init, const double* trans, int64_t B, int32_t n, int32_t m,
                                double* logz, double* marg_init, double* marg_trans, int32_t* status,
                                void* workspace, size_t ws_bytes, void* stream) {
  if (B < 0 || n < 1 || m < 1 || !init || (n > 1 && !trans) || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!workspace || ws_bytes < sdb_chain_fb_f64_workspace(B, n, m)) return SDB_ERR_WORKSPACE;
  chain_exact_kernel<<<(unsigned)B, kT, 0, (cudaStream_t)stream>>>(init, trans, n, m, (double*)workspace, logz,
                                                                    marg_init, marg_trans, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" size_t sdb_semimarkov_fb_f64_workspace(int64_t B, int32_t n, int32_t s, int32_t m) {
  (void)s;
  return (B < 0 || n < 1 || m < 1) ? 0 : (size_t)B * 2 * (n + 1) * m * sizeof(double) + 256;
}
// chain.py:250-298 in fp64: segment_potentials [B,n,s,m,m] float64; marg nullable
extern "C" int sdb_semimarkov_fb_f64(const double* segment_potentials, int64_t B, int32_t n, int32_t s, int32_t m,
                                     double* logz, double* marg, int32_t* status, void* workspace, size_t ws_bytes,
                                     void* stream) {
  if (B < 0 || n < 1 || s < 1 || m < 1 || !segment_potentials || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!workspace || ws_bytes < sdb_semimarkov_fb_f64_workspace(B, n, s, m)) return SDB_ERR_WORKSPACE;
  semimarkov_exact_kernel<<<(unsigned)B, kT, 0, (cudaStream_t)stream>>>(segment_potentials, n, s, m,
                                                                         (double*)workspace, logz, marg, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
