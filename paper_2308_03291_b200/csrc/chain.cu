// Linear-chain CRF: forward-backward (log semiring) and Viterbi (max-plus).
//
// Reference: structdist chain.py:64-114 (_forward, _backward,
// forward_log_partition, chain_marginals, chain_argmax).
//
// Layout (per instance b): init [m], trans [n-1][m][m] (step, prev, next),
// fp32, contiguous, batch-major.
//
// Forward/backward: one CTA per (instance, direction).  Each step is an
// m x m log-semiring mat-vec; the vector is renormalised every step by its
// max (c_t), so stored alpha~/beta~ are <= 0 and small; the cumulative
// normalisers are kept in fp64 (fp32 log-space without
// normalisation is at the 1e-4 edge at n=128).  Marginals are a streaming
// pass exp(alpha~_t[a] + theta_t[a,b] + beta~_{t+1}[b] + K_t) with
// K_t = A_t + B_{t+1} - logZ folded in fp64.
//
// Viterbi runs in fp64 with the reference's addition order
// (score[a] + theta[a,b]) so argmax ties and sums are bit-identical to the
// float64 reference on the same fp32 inputs.
#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kGroups = kThreads / 32;  // row groups for the column reduce

struct ChainWs {
  float* alpha;   // [B][n][m] normalised forward
  float* beta;    // [B][n][m] normalised backward
  double* acum;   // [B][n] cumulative forward normalisers
  double* bcum;   // [B][n] cumulative backward normalisers
  int32_t* flags; // [B] forward status
};

__host__ ChainWs carve_chain(void* base, int64_t B, int n, int m, size_t* bytes) {
  Carve c(base);
  ChainWs w;
  w.alpha = c.take<float>((size_t)B * n * m);
  w.beta = c.take<float>((size_t)B * n * m);
  w.acum = c.take<double>((size_t)B * n);
  w.bcum = c.take<double>((size_t)B * n);
  w.flags = c.take<int32_t>((size_t)B);
  *bytes = c.used;
  return w;
}

// block-wide max of one float per thread; `red` holds kThreads/32 floats
__device__ float block_max(float v, float* red) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  float r = red[0];
#pragma unroll
  for (int i = 1; i < kThreads / 32; ++i) r = fmaxf(r, red[i]);
  __syncthreads();
  return r;
}

__device__ int block_or(int v, int* red) {
  v = __any_sync(0xffffffffu, v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  int r = 0;
#pragma unroll
  for (int i = 0; i < kThreads / 32; ++i) r |= red[i];
  __syncthreads();
  return r;
}

// grid (B, 2): y == 0 forward, y == 1 backward
__global__ void __launch_bounds__(kThreads) chain_fwd_bwd_kernel(
    const float* __restrict__ init, const float* __restrict__ trans, int n, int m, ChainWs ws,
    double* __restrict__ logz, int32_t* __restrict__ status) {
  extern __shared__ float sm[];
  float* vec = sm;                       // [m]   current normalised vector
  float* pm = vec + m;                   // [kGroups][m] partial max
  float* ps = pm + kGroups * m;          // [kGroups][m] partial sum
  __shared__ float redf[kThreads / 32];
  __shared__ int redi[kThreads / 32];

  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t mm = (size_t)m * m;
  const float* th = trans + (size_t)b * (n - 1) * mm;
  int bad = 0;

  if (blockIdx.y == 0) {
    // ---------------- forward: alpha_{t+1}[j] = lse_a alpha_t[a] + th_t[a][j]
    float* al = ws.alpha + (size_t)b * n * m;
    double* ac = ws.acum + (size_t)b * n;
    float lmax = ninf();
    for (int j = tid; j < m; j += kThreads) {
      float x = init[(size_t)b * m + j];
      bad |= bad_input(x);
      vec[j] = x;
      lmax = fmaxf(lmax, x);
    }
    float c = block_max(lmax, redf);
    bool vac = (c == ninf());
    double A = vac ? 0.0 : (double)c;
    if (vac) c = 0.f;
    for (int j = tid; j < m; j += kThreads) {
      vec[j] -= c;
      al[j] = vec[j];
    }
    if (tid == 0) ac[0] = A;
    __syncthreads();
    for (int t = 0; t < n - 1 && !vac; ++t) {
      const float* tt = th + (size_t)t * mm;
      // phase 1: partial column lse over row groups
      for (int j0 = 0; j0 < m; j0 += 32) {
        const int j = j0 + lane;
        if (j < m) {
          Lse acc;
          for (int a = warp; a < m; a += kGroups) {
            float x = tt[(size_t)a * m + j];
            bad |= bad_input(x);
            acc.add(vec[a] + x);
          }
          pm[warp * m + j] = acc.m;
          ps[warp * m + j] = acc.s;
        }
      }
      __syncthreads();
      // phase 2: merge groups -> u_j, block max
      float u[4];
      float lm = ninf();
      int q = 0;
      for (int j = tid; j < m; j += kThreads, ++q) {
        Lse acc;
#pragma unroll
        for (int g = 0; g < kGroups; ++g) acc.merge(pm[g * m + j], ps[g * m + j]);
        float r = acc.result();
        if (q < 4) u[q] = r;
        lm = fmaxf(lm, r);
      }
      c = block_max(lm, redf);  // (contains __syncthreads)
      if (c == ninf()) {
        vac = true;
        break;
      }
      A += (double)c;
      q = 0;
      for (int j = tid; j < m; j += kThreads, ++q) {
        float v = u[q] - c;
        vec[j] = v;
        al[(size_t)(t + 1) * m + j] = v;
      }
      if (tid == 0) ac[t + 1] = A;
      __syncthreads();
    }
    bad = block_or(bad, redi);
    // logZ = A + lse(alpha~_{n-1})
    if (!vac) {
      float lm = ninf();
      for (int j = tid; j < m; j += kThreads) lm = fmaxf(lm, vec[j]);
      float mx = block_max(lm, redf);
      float s = 0.f;
      for (int j = tid; j < m; j += kThreads) s += fexp(vec[j] - mx);
      s = warp_sum(s);
      if (lane == 0) redf[warp] = s;
      __syncthreads();
      if (tid == 0) {
        float tot = 0.f;
        for (int i = 0; i < kThreads / 32; ++i) tot += redf[i];
        double z = A + (double)mx + (double)flog(tot);
        logz[b] = z;
      }
    } else if (tid == 0) {
      logz[b] = ninfd();
    }
    if (tid == 0) {
      int st = bad ? SDB_ST_INVALID : (vac ? SDB_ST_VACUOUS : SDB_ST_OK);
      status[b] = st;
      ws.flags[b] = st;
    }
  } else {
    // ---------------- backward: beta_t[a] = lse_j th_t[a][j] + beta_{t+1}[j]
    float* be = ws.beta + (size_t)b * n * m;
    double* bc = ws.bcum + (size_t)b * n;
    for (int j = tid; j < m; j += kThreads) {
      vec[j] = 0.f;
      be[(size_t)(n - 1) * m + j] = 0.f;
    }
    double Bc = 0.0;
    if (tid == 0) bc[n - 1] = 0.0;
    __syncthreads();
    for (int t = n - 2; t >= 0; --t) {
      const float* tt = th + (size_t)t * mm;
      float lm = ninf();
      for (int a = warp; a < m; a += kGroups) {
        Lse acc;
        for (int j = lane; j < m; j += 32) acc.add(tt[(size_t)a * m + j] + vec[j]);
        // warp merge
        float mx = warp_max(acc.m);
        float s = (mx == ninf()) ? 0.f : acc.s * fexp(acc.m - mx);
        s = warp_sum(s);
        float r = (mx == ninf()) ? ninf() : mx + flog(s);
        if (lane == 0) pm[a] = r;
        lm = fmaxf(lm, r);
      }
      float d = block_max(lm, redf);  // syncs: pm visible
      if (d == ninf()) d = 0.f;
      Bc += (double)d;
      for (int a = tid; a < m; a += kThreads) {
        float v = pm[a] - d;
        vec[a] = v;
        be[(size_t)t * m + a] = v;
      }
      if (tid == 0) bc[t] = Bc;
      __syncthreads();
    }
  }
}

// marginals: grid (ceil((n-1)/kStepsPerBlock) + 1, B).  blockIdx.x == 0 also
// writes p_init.
constexpr int kStepsPerBlock = 8;

__global__ void __launch_bounds__(kThreads) chain_marg_kernel(
    const float* __restrict__ init, const float* __restrict__ trans, int n, int m, ChainWs ws,
    const double* __restrict__ logz, float* __restrict__ marg_init, float* __restrict__ marg_trans) {
  const int b = blockIdx.y;
  const int t0 = blockIdx.x * kStepsPerBlock;
  const size_t mm = (size_t)m * m;
  const bool ok = ws.flags[b] == SDB_ST_OK;
  const double z = logz[b];
  if (blockIdx.x == 0 && marg_init) {
    const float* be = ws.beta + (size_t)b * n * m;
    float K = ok ? (float)(ws.bcum[(size_t)b * n] - z) : 0.f;
    for (int j = threadIdx.x; j < m; j += kThreads)
      marg_init[(size_t)b * m + j] = ok ? fexp(init[(size_t)b * m + j] + be[j] + K) : 0.f;
  }
  if (!marg_trans) return;
  const int t1 = min(t0 + kStepsPerBlock, n - 1);
  for (int t = t0; t < t1; ++t) {
    const float* tt = trans + ((size_t)b * (n - 1) + t) * mm;
    float* out = marg_trans + ((size_t)b * (n - 1) + t) * mm;
    if (!ok) {
      for (size_t e = threadIdx.x; e < mm; e += kThreads) out[e] = 0.f;
      continue;
    }
    const float* al = ws.alpha + ((size_t)b * n + t) * m;
    const float* be = ws.beta + ((size_t)b * n + t + 1) * m;
    const float K = (float)(ws.acum[(size_t)b * n + t] + ws.bcum[(size_t)b * n + t + 1] - z);
    if ((m & 3) == 0) {
      const float4* t4 = reinterpret_cast<const float4*>(tt);
      float4* o4 = reinterpret_cast<float4*>(out);
      const int m4 = m >> 2;
      for (int e = threadIdx.x; e < (int)(mm >> 2); e += kThreads) {
        const int a = e / m4, j = (e - a * m4) * 4;
        const float x = al[a] + K;
        float4 v = __ldg(t4 + e);
        float4 r;
        r.x = fexp(x + v.x + be[j + 0]);
        r.y = fexp(x + v.y + be[j + 1]);
        r.z = fexp(x + v.z + be[j + 2]);
        r.w = fexp(x + v.w + be[j + 3]);
        o4[e] = r;
      }
    } else {
      for (int e = threadIdx.x; e < (int)mm; e += kThreads) {
        const int a = e / m, j = e - a * m;
        out[e] = fexp(al[a] + tt[e] + be[j] + K);
      }
    }
  }
}

// ---------------------------------------------------------------- Viterbi
// grid B; fp64 scores; backpointers uint16 in smem (or workspace if large).
__global__ void __launch_bounds__(kThreads) chain_viterbi_kernel(
    const float* __restrict__ init, const float* __restrict__ trans, int n, int m,
    uint16_t* __restrict__ gback, int back_in_smem, int32_t* __restrict__ tags,
    double* __restrict__ score, int32_t* __restrict__ status) {
  extern __shared__ double smd[];
  double* sc = smd;                      // [m]
  double* pv = sc + m;                   // [kGroups][m]
  int* pa = (int*)(pv + kGroups * m);    // [kGroups][m]
  uint16_t* back = back_in_smem ? (uint16_t*)(pa + kGroups * m) : gback + (size_t)blockIdx.x * n * m;
  __shared__ int redi[kThreads / 32];
  __shared__ double bestv[kThreads / 32];
  __shared__ int besti[kThreads / 32];

  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t mm = (size_t)m * m;
  const float* th = trans + (size_t)b * (n - 1) * mm;
  int bad = 0;
  for (int j = tid; j < m; j += kThreads) {
    float x = init[(size_t)b * m + j];
    bad |= bad_input(x);
    sc[j] = (double)x;
  }
  __syncthreads();
  for (int t = 0; t < n - 1; ++t) {
    const float* tt = th + (size_t)t * mm;
    for (int j0 = 0; j0 < m; j0 += 32) {
      const int j = j0 + lane;
      if (j < m) {
        double best = ninfd();
        int arg = 0x7fffffff;
        for (int a = warp; a < m; a += kGroups) {
          float x = tt[(size_t)a * m + j];
          bad |= bad_input(x);
          double v = sc[a] + (double)x;
          if (v > best || (v == best && a < arg)) {
            best = v;
            arg = a;
          }
        }
        pv[warp * m + j] = best;
        pa[warp * m + j] = arg;
      }
    }
    __syncthreads();
    for (int j = tid; j < m; j += kThreads) {
      double best = pv[j];
      int arg = pa[j];
#pragma unroll
      for (int g = 1; g < kGroups; ++g) {
        double v = pv[g * m + j];
        int a = pa[g * m + j];
        if (v > best || (v == best && a < arg)) {
          best = v;
          arg = a;
        }
      }
      sc[j] = best;
      back[(size_t)(t + 1) * m + j] = (uint16_t)arg;
    }
    __syncthreads();
  }
  bad = block_or(bad, redi);
  // final first-argmax
  double best = ninfd();
  int arg = 0x7fffffff;
  for (int j = tid; j < m; j += kThreads) {
    double v = sc[j];
    if (v > best || (v == best && j < arg)) {
      best = v;
      arg = j;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oa = __shfl_xor_sync(0xffffffffu, arg, o);
    if (ov > best || (ov == best && oa < arg)) {
      best = ov;
      arg = oa;
    }
  }
  if (lane == 0) {
    bestv[warp] = best;
    besti[warp] = arg;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kThreads / 32; ++w) {
      if (bestv[w] > best || (bestv[w] == best && besti[w] < arg)) {
        best = bestv[w];
        arg = besti[w];
      }
    }
    int32_t* tg = tags + (size_t)b * n;
    const bool vac = (best == ninfd());
    status[b] = bad ? SDB_ST_INVALID : (vac ? SDB_ST_VACUOUS : SDB_ST_OK);
    score[b] = best;
    int cur = vac ? 0 : arg;
    tg[n - 1] = cur;
    for (int t = n - 2; t >= 0; --t) {
      cur = vac ? 0 : back[(size_t)(t + 1) * m + cur];
      tg[t] = cur;
    }
  }
}

size_t viterbi_smem(int n, int m, bool with_back) {
  size_t s = (size_t)m * 8 + (size_t)kGroups * m * 12;
  if (with_back) s += (size_t)n * m * 2;
  return s;
}

}  // namespace

extern "C" size_t sdb_chain_fb_workspace(int64_t B, int32_t n, int32_t m) {
  size_t bytes = 0;
  carve_chain(nullptr, B, n, m, &bytes);
  return bytes;
}

extern "C" int sdb_chain_fb(const float* init, const float* trans, int64_t B, int32_t n, int32_t m,
                            double* logz, float* marg_init, float* marg_trans, int32_t* status,
                            void* workspace, size_t ws_bytes, void* stream) {
  if (B < 0 || n < 1 || m < 1 || m > 1024 || !init || (n > 1 && !trans) || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  size_t need = 0;
  ChainWs ws = carve_chain(workspace, B, n, m, &need);
  if (!workspace || ws_bytes < need) return SDB_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  size_t smem = (size_t)m * 4 * (1 + 2 * kGroups);
  if (smem > 48 * 1024) {
    if (cudaFuncSetAttribute(chain_fwd_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SDB_ERR_CUDA;
  }
  chain_fwd_bwd_kernel<<<dim3((unsigned)B, 2), kThreads, smem, s>>>(init, trans, n, m, ws, logz, status);
  SDB_CHECK_LAUNCH();
  if (marg_init || marg_trans) {
    dim3 g((unsigned)((n - 1 + kStepsPerBlock - 1) / kStepsPerBlock + (n == 1 ? 1 : 0)), (unsigned)B);
    chain_marg_kernel<<<g, kThreads, 0, s>>>(init, trans, n, m, ws, logz, marg_init, marg_trans);
    SDB_CHECK_LAUNCH();
  }
  return SDB_OK;
}

extern "C" size_t sdb_chain_viterbi_workspace(int64_t B, int32_t n, int32_t m) {
  if (viterbi_smem(n, m, true) <= 160 * 1024) return 256;
  return (size_t)B * n * m * sizeof(uint16_t) + 256;
}

extern "C" int sdb_chain_viterbi(const float* init, const float* trans, int64_t B, int32_t n, int32_t m,
                                 int32_t* tags, double* score, int32_t* status, void* workspace,
                                 size_t ws_bytes, void* stream) {
  if (B < 0 || n < 1 || m < 1 || m > 1024 || !init || (n > 1 && !trans) || !tags || !score || !status)
    return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!workspace || ws_bytes < sdb_chain_viterbi_workspace(B, n, m)) return SDB_ERR_WORKSPACE;
  const bool in_smem = viterbi_smem(n, m, true) <= 160 * 1024;
  size_t smem = viterbi_smem(n, m, in_smem);
  if (smem > 48 * 1024) {
    if (cudaFuncSetAttribute(chain_viterbi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SDB_ERR_CUDA;
  }
  chain_viterbi_kernel<<<(unsigned)B, kThreads, smem, (cudaStream_t)stream>>>(
      init, trans, n, m, (uint16_t*)workspace, in_smem ? 1 : 0, tags, score, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
