// Semi-Markov CRF (segmental chain): log-partition, segment marginals,
// segmental Viterbi.
//
// Reference: structdist chain.py:250-327 (_sm_forward, _sm_backward,
// semi_markov_log_partition, semi_markov_marginals, semi_markov_argmax).
// Layout per instance: segment_potentials [n][s][m][m] fp32 indexed
// (segment start, width-1, previous label, label); virtual start label 0.
//
// One CTA (256 threads) per instance.  alpha [n+1][m] and beta [n+1][m] are
// fp64 in shared memory (n*m small for this family); each position is a
// log-semiring contraction over (width, previous label) computed by
// thread groups over p with a fixed-order merge.  Marginals are a streaming
// pass over the [n][s][m][m] output (zeros where t + w > n).  Viterbi is fp64
// in the reference's scan order (w ascending, first argmax over p, strict '>').
#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kGroups = kThreads / 32;

size_t sm_smem(int n, int m) { return (size_t)2 * (n + 1) * m * 8 + (size_t)2 * kGroups * m * 8 + 64; }

template <int kMode>  // 0 logZ, 1 logZ + marginals
__global__ void __launch_bounds__(kThreads) semimarkov_kernel(const float* __restrict__ th_all, int n, int s, int m,
                                                              double* __restrict__ logz, float* __restrict__ marg_all,
                                                              int32_t* __restrict__ status) {
  extern __shared__ __align__(16) double smd[];
  double* al = smd;                  // [n+1][m]
  double* be = al + (size_t)(n + 1) * m;
  double* pm = be + (size_t)(n + 1) * m;  // [kGroups][m] partial max
  float* ps = (float*)(pm + kGroups * m); // [kGroups][m] partial sum
  __shared__ int badsh;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t mm = (size_t)m * m;
  const float* th = th_all + (size_t)b * n * s * mm;
  if (tid == 0) badsh = 0;
  {
    int bad = 0;
    for (size_t e = tid; e < (size_t)n * s * mm; e += kThreads) bad |= bad_input(th[e]);
    if (bad) atomicOr(&badsh, 1);
  }
  for (int l = tid; l < m; l += kThreads) al[l] = (l == 0) ? 0.0 : ninfd();
  __syncthreads();
  // ---- forward (chain.py:250-265): alpha[t][l] = lse_{w,p} alpha[t-w][p] + th[t-w][w-1][p][l]
  for (int t = 1; t <= n; ++t) {
    for (int l0 = 0; l0 < m; l0 += 32) {
      const int l = l0 + lane;
      double mx = ninfd();
      float sum = 0.f;
      if (l < m) {
        for (int w = 1; w <= min(s, t); ++w) {
          const float* tt = th + ((size_t)(t - w) * s + (w - 1)) * mm;
          for (int p = warp; p < m; p += kGroups) {
            const double x = al[(size_t)(t - w) * m + p] + (double)tt[(size_t)p * m + l];
            if (x > mx) { sum = sum * fexp((float)(mx - x)) + 1.f; mx = x; }
            else if (x != ninfd()) sum += fexp((float)(x - mx));
          }
        }
        pm[warp * m + l] = mx;
        ps[warp * m + l] = sum;
      }
    }
    __syncthreads();
    for (int l = tid; l < m; l += kThreads) {
      LseD acc;
      for (int g = 0; g < kGroups; ++g) acc.merge(pm[g * m + l], ps[g * m + l]);
      al[(size_t)t * m + l] = acc.result();
    }
    __syncthreads();
  }
  __shared__ double zsh;
  if (tid == 0) {
    LseD acc;
    for (int l = 0; l < m; ++l) acc.add(al[(size_t)n * m + l]);
    zsh = acc.result();
    const int st = badsh ? SDB_ST_INVALID : (zsh == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
    status[b] = st;
    logz[b] = zsh;
  }
  __syncthreads();
  if (kMode == 0) return;
  const double Z = zsh;
  float* mg = marg_all + (size_t)b * n * s * mm;
  if (Z == ninfd() || badsh) {
    for (size_t e = tid; e < (size_t)n * s * mm; e += kThreads) mg[e] = 0.f;
    return;
  }
  // ---- backward (chain.py:272-282): beta[t][p] = lse_{w,l} th[t][w-1][p][l] + beta[t+w][l]
  for (int p = tid; p < m; p += kThreads) be[(size_t)n * m + p] = 0.0;
  __syncthreads();
  for (int t = n - 1; t >= 0; --t) {
    for (int p = warp; p < m; p += kGroups) {
      LseD acc;
      for (int w = 1; w <= min(s, n - t); ++w) {
        const float* tt = th + ((size_t)t * s + (w - 1)) * mm + (size_t)p * m;
        for (int l = lane; l < m; l += 32) acc.add((double)tt[l] + be[(size_t)(t + w) * m + l]);
      }
      // warp merge
      double M = warp_maxd(acc.m);
      float e = (M == ninfd() || acc.m == ninfd()) ? 0.f : acc.s * fexp((float)(acc.m - M));
      e = warp_sum(e);
      if (lane == 0) be[(size_t)t * m + p] = (M == ninfd()) ? ninfd() : M + (double)flog(e);
    }
    __syncthreads();
  }
  // ---- marginals (chain.py:285-298)
  const size_t tot = (size_t)n * s * mm;
  for (size_t e = tid; e < tot; e += kThreads) {
    const size_t ts = e / mm;
    const int t = (int)(ts / s), w = (int)(ts - (size_t)t * s) + 1;
    const int r = (int)(e - ts * mm), p = r / m, l = r - p * m;
    float v = 0.f;
    if (t + w <= n) {
      const double a = al[(size_t)t * m + p], bb = be[(size_t)(t + w) * m + l];
      if (a != ninfd() && bb != ninfd()) v = fexp((float)(a + bb - Z) + th[e]);
    }
    mg[e] = v;
  }
}

// ------------------------------------------------------------- Viterbi
// score/back in global workspace; thread per label, fp64, reference order.
__global__ void semimarkov_viterbi_kernel(const float* __restrict__ th_all, int n, int s, int m,
                                          double* __restrict__ sc_all, int32_t* __restrict__ back_all,
                                          int32_t* __restrict__ seg_all, int32_t* __restrict__ nseg,
                                          double* __restrict__ score, int32_t* __restrict__ status) {
  const int b = blockIdx.x, tid = threadIdx.x;
  const size_t mm = (size_t)m * m;
  const float* th = th_all + (size_t)b * n * s * mm;
  double* sc = sc_all + (size_t)b * (n + 1) * m;
  int32_t* back = back_all + (size_t)b * (n + 1) * m;  // (w << 16) | p, -1 none
  __shared__ int badsh;
  if (tid == 0) badsh = 0;
  __syncthreads();
  {
    int bad = 0;
    for (size_t e = tid; e < (size_t)n * s * mm; e += blockDim.x) bad |= bad_input(th[e]);
    if (bad) atomicOr(&badsh, 1);
  }
  for (int l = tid; l < m; l += blockDim.x) sc[l] = (l == 0) ? 0.0 : ninfd();
  __syncthreads();
  for (int t = 1; t <= n; ++t) {
    for (int l = tid; l < m; l += blockDim.x) {
      double best = ninfd();
      int arg = -1;
      for (int w = 1; w <= min(s, t); ++w) {
        const float* tt = th + ((size_t)(t - w) * s + (w - 1)) * mm;
        // first argmax over p of sc[t-w][p] + th[t-w][w-1][p][l]
        double cb = ninfd();
        int cp = 0;
        for (int p = 0; p < m; ++p) {
          const double x = sc[(size_t)(t - w) * m + p] + (double)tt[(size_t)p * m + l];
          if (x > cb) { cb = x; cp = p; }
        }
        if (cb > best) { best = cb; arg = (w << 16) | cp; }
      }
      sc[(size_t)t * m + l] = best;
      back[(size_t)t * m + l] = arg;
    }
    __syncthreads();
  }
  if (tid == 0) {
    double best = ninfd();
    int l = 0;
    for (int q = 0; q < m; ++q)
      if (sc[(size_t)n * m + q] > best) { best = sc[(size_t)n * m + q]; l = q; }
    const int st = badsh ? SDB_ST_INVALID : (best == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
    status[b] = st;
    score[b] = best;
    int32_t* seg = seg_all + (size_t)b * n * 4;
    int cnt = 0;
    if (st == SDB_ST_OK) {
      // walk back (chain.py:318-325), then reverse into (start, width, prev, label)
      int t = n;
      while (t > 0) {
        const int code = back[(size_t)t * m + l];
        const int w = code >> 16, p = code & 0xffff;
        seg[4 * cnt + 0] = t - w;
        seg[4 * cnt + 1] = w;
        seg[4 * cnt + 2] = p;
        seg[4 * cnt + 3] = l;
        ++cnt;
        t -= w;
        l = p;
      }
      for (int a = 0, z = cnt - 1; a < z; ++a, --z)
        for (int q = 0; q < 4; ++q) {
          const int tmp = seg[4 * a + q];
          seg[4 * a + q] = seg[4 * z + q];
          seg[4 * z + q] = tmp;
        }
    }
    nseg[b] = cnt;
  }
}

int sm_check(int64_t B, int n, int s, int m) {
  if (B < 0 || n < 1 || s < 1 || s > n || m < 1) return SDB_ERR_ARG;
  if (sm_smem(n, m) > 200 * 1024 || m > 65535) return SDB_ERR_UNSUPPORTED;
  return SDB_OK;
}

}  // namespace

extern "C" int sdb_semimarkov_fb(const float* segment_potentials, int64_t B, int32_t n, int32_t s, int32_t m,
                                 double* logz, float* marg, int32_t* status, void* stream) {
  int rc = sm_check(B, n, s, m);
  if (rc) return rc;
  if (!segment_potentials || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  const size_t smem = sm_smem(n, m);
  cudaStream_t st = (cudaStream_t)stream;
  if (marg) {
    if (sdb_set_smem((const void*)semimarkov_kernel<1>, smem) != cudaSuccess)
      return SDB_ERR_CUDA;
    semimarkov_kernel<1><<<(unsigned)B, kThreads, smem, st>>>(segment_potentials, n, s, m, logz, marg, status);
  } else {
    if (sdb_set_smem((const void*)semimarkov_kernel<0>, smem) != cudaSuccess)
      return SDB_ERR_CUDA;
    semimarkov_kernel<0><<<(unsigned)B, kThreads, smem, st>>>(segment_potentials, n, s, m, logz, nullptr, status);
  }
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" size_t sdb_semimarkov_viterbi_workspace(int64_t B, int32_t n, int32_t s, int32_t m) {
  (void)s;
  return (size_t)B * (n + 1) * m * (8 + 4) + 512;
}

extern "C" int sdb_semimarkov_viterbi(const float* segment_potentials, int64_t B, int32_t n, int32_t s, int32_t m,
                                      int32_t* segments, int32_t* num_segments, double* score, int32_t* status,
                                      void* workspace, size_t ws_bytes, void* stream) {
  int rc = sm_check(B, n, s, m);
  if (rc) return rc;
  if (!segment_potentials || !segments || !num_segments || !score || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!workspace || ws_bytes < sdb_semimarkov_viterbi_workspace(B, n, s, m)) return SDB_ERR_WORKSPACE;
  Carve c(workspace);
  double* sc = c.take<double>((size_t)B * (n + 1) * m);
  int32_t* back = c.take<int32_t>((size_t)B * (n + 1) * m);
  semimarkov_viterbi_kernel<<<(unsigned)B, 128, 0, (cudaStream_t)stream>>>(segment_potentials, n, s, m, sc, back,
                                                                           segments, num_segments, score, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
