// Span-factored Tree-CRF (CKY): log-partition, labeled-span marginals,
// max-plus argmax.
//
// Reference: structdist constituency.py:52-133 (_tree_charts,
// cky_log_partition, tree_marginals, _tree_walk, tree_argmax).
// Layout per instance: span_potentials [n][n][m] fp32 (only i <= j is read;
// marginals for i > j are written as 0).
//
// One CTA per instance (kThreads threads, kWarps warps):
//   1. label fold: fold[i,j] = lse_l theta[i,j,l] -- one warp per span, the
//      32 lanes read the contiguous label row (coalesced), warp lse;
//   2. inside by span width (constituency.py:57-63): one warp per cell of the
//      current width, lanes over split points, warp lse; one barrier/width;
//   3. outside by decreasing width (constituency.py:84-99): lanes over the
//      n-w parent terms (right-sibling then left-sibling parents);
//   4. marginals: exp(outside + inside - fold + theta - Z) streamed over the
//      full [n][n][m] output with 16-byte stores.
// Charts are packed upper-triangular in shared memory, fp64 (inside values
// grow to ~n*log(m*4)); exp/log in fp32 MUFU on differences.
#include "common.cuh"

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ int tri(int i, int j, int n) { return i * n - (i * (i - 1)) / 2 + (j - i); }

size_t tree_smem(int n) {
  const size_t T = (size_t)n * (n + 1) / 2;
  return T * 8 * 2 + T * 4 + 64;
}

// warp-wide lse of per-lane (max, sum) partials over doubles.  The common
// shift only has to be CLOSE to the max (the partial sums are rescaled by
// exp(m - M) <= ~1), so it is reduced in fp32 (one shuffle per round instead
// of two + a double compare) and the result stays exact in fp64.
__device__ __forceinline__ double warp_lse_d(double m, float s) {
  const float mf = warp_max((float)m);
  const double M = (double)mf;
  float e = (mf == ninf() || m == ninfd()) ? 0.f : s * fexp((float)(m - M));
  e = warp_sum(e);
  return (mf == ninf()) ? ninfd() : M + (double)flog(e);
}

template <int kMode>  // 0 logZ, 1 logZ+marginals, 2 max-plus argmax
__global__ void __launch_bounds__(kThreads) tree_kernel(const float* __restrict__ th_all, int n, int m,
                                                         double* __restrict__ logz, float* __restrict__ marg_all,
                                                         int32_t* __restrict__ labels_all,
                                                         double* __restrict__ score, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) char smraw[];
  const size_t T = (size_t)n * (n + 1) / 2;
  double* ins = (double*)smraw;
  double* out = ins + T;
  float* fold = (float*)(out + T);
  __shared__ int badsh;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* th = th_all + (size_t)b * n * n * m;
  if (tid == 0) badsh = 0;
  __syncthreads();
  constexpr bool kMax = (kMode == 2);

  // ---- 1. label fold over the upper triangle (constituency.py:55): thread per
  // span, the label row read with 16-byte loads all in flight at once (a warp
  // per span was latency-bound on one dependent global load per span)
  int bad = 0;
  const bool vec4 = ((m & 3) == 0) && ((((uintptr_t)th) & 15) == 0);
  for (int idx = tid; idx < (int)T; idx += kThreads) {
    // map packed index -> (i, j): row i starts at tri(i, i) = i n - i (i-1) / 2
    const float b2 = 2.f * n + 1.f;
    int i = (int)((b2 - sqrtf(b2 * b2 - 8.f * idx)) * 0.5f);
    i = max(0, min(i, n - 1));
    while (i > 0 && tri(i, i, n) > idx) --i;
    while (i + 1 < n && tri(i + 1, i + 1, n) <= idx) ++i;
    const int j = i + (idx - tri(i, i, n));
    const float* row = th + ((size_t)i * n + j) * m;
    float mx = ninf(), sm = 0.f;
    // online (max, sum): one pass over the row
    auto add = [&](float x) {
      bad |= bad_input(x);
      if (kMax) {
        mx = fmaxf(mx, x);
      } else if (x > mx) {
        sm = (mx == ninf()) ? 1.f : sm * fexp(mx - x) + 1.f;
        mx = x;
      } else if (x != ninf()) {
        sm += fexp(x - mx);
      }
    };
    if (vec4) {
      const float4* r4 = reinterpret_cast<const float4*>(row);
      int l4 = 0;
      for (; l4 + 8 <= m / 4; l4 += 8) {
        float4 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = __ldg(r4 + l4 + q);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          add(v[q].x);
          add(v[q].y);
          add(v[q].z);
          add(v[q].w);
        }
      }
      for (; l4 < m / 4; ++l4) {
        const float4 v = __ldg(r4 + l4);
        add(v.x);
        add(v.y);
        add(v.z);
        add(v.w);
      }
    } else {
      for (int l = 0; l < m; ++l) add(__ldg(row + l));
    }
    fold[idx] = kMax ? mx : ((mx == ninf()) ? ninf() : mx + flog(sm));
  }
  if (bad) atomicOr(&badsh, 1);
  __syncthreads();

  // ---- 2. inside (width 1 = fold; width w: fold + lse_k ins[i,k] + ins[k+1,j])
  for (int i = tid; i < n; i += kThreads) ins[tri(i, i, n)] = (double)fold[tri(i, i, n)];
  __syncthreads();
  for (int w = 2; w <= n; ++w) {
    for (int i = warp; i <= n - w; i += kWarps) {
      const int j = i + w - 1;
      double r;
      // each lane holds <= 4 split terms (n <= 128): read them once
      double t[4];
      double mloc = ninfd();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = i + lane + 32 * q;
        t[q] = (k < j) ? ins[tri(i, k, n)] + ins[tri(k + 1, j, n)] : ninfd();
        mloc = fmax(mloc, t[q]);
      }
      if (kMax) {
        r = warp_maxd(mloc);
      } else {
        float s = 0.f;
        if (mloc != ninfd())
#pragma unroll
          for (int q = 0; q < 4; ++q) s += (t[q] == ninfd()) ? 0.f : fexp((float)(t[q] - mloc));
        r = warp_lse_d(mloc, s);
      }
      if (lane == 0) {
        const float f = fold[tri(i, j, n)];
        ins[tri(i, j, n)] = (r == ninfd() || f == ninf()) ? ninfd() : (double)f + r;
      }
    }
    __syncthreads();
  }
  const double Z = ins[tri(0, n - 1, n)];
  const bool zok = Z != ninfd();

  if (kMode == 0 || (kMode == 1 && !zok) || (kMode == 2 && !zok)) {
    if (tid == 0) {
      status[b] = badsh ? SDB_ST_INVALID : (zok ? SDB_ST_OK : SDB_ST_VACUOUS);
      if (kMode == 2) score[b] = Z; else logz[b] = Z;
    }
    if (kMode == 1) {  // vacuous: zero marginals
      float4* o4 = reinterpret_cast<float4*>(marg_all + (size_t)b * n * n * m);
      const size_t tot = (size_t)n * n * m;
      if ((tot & 3) == 0 && ((uintptr_t)o4 & 15) == 0)
        for (size_t e = tid; e < tot / 4; e += kThreads) o4[e] = make_float4(0.f, 0.f, 0.f, 0.f);
      else
        for (size_t e = tid; e < tot; e += kThreads) marg_all[(size_t)b * n * n * m + e] = 0.f;
    }
    if (kMode == 2 && tid == 0 && !zok) {
      int32_t* lab = labels_all + (size_t)b * n * n;
      for (int e = 0; e < n * n; ++e) lab[e] = -1;
    }
    return;
  }

  if (kMode == 2) {
    // ---- top-down walk (constituency.py:113-126) by warp 0; explicit stack in `out`
    if (warp == 0) {
      int32_t* lab = labels_all + (size_t)b * n * n;
      for (int e = lane; e < n * n; e += 32) lab[e] = -1;
      __syncwarp();
      int* stk = (int*)out;  // pairs (i, j)
      int sp = 0;
      if (lane == 0) { stk[0] = 0; stk[1] = n - 1; }
      sp = 1;
      while (sp > 0) {
        __syncwarp();
        const int i = stk[2 * (sp - 1)], j = stk[2 * (sp - 1) + 1];
        --sp;
        // label = first argmax over theta[i,j,:]
        const float* row = th + ((size_t)i * n + j) * m;
        float bv = ninf();
        int bl = 0x7fffffff;
        for (int l = lane; l < m; l += 32) {
          const float x = row[l];
          if (x > bv || (x == bv && l < bl)) { bv = x; bl = l; }
        }
        for (int o = 16; o > 0; o >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
          if (ov > bv || (ov == bv && ol < bl)) { bv = ov; bl = ol; }
        }
        if (bl == 0x7fffffff) bl = 0;
        if (lane == 0) lab[(size_t)i * n + j] = bl;
        if (i != j) {
          double kv = ninfd();
          int kk = 0x7fffffff;
          for (int k = i + lane; k < j; k += 32) {
            const double v = ins[tri(i, k, n)] + ins[tri(k + 1, j, n)];
            if (v > kv || (v == kv && k < kk)) { kv = v; kk = k; }
          }
          for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, kv, o);
            const int ok = __shfl_xor_sync(0xffffffffu, kk, o);
            if (ov > kv || (ov == kv && ok < kk)) { kv = ov; kk = ok; }
          }
          if (kk == 0x7fffffff) kk = i;
          __syncwarp();
          if (lane == 0) {
            stk[2 * sp] = i; stk[2 * sp + 1] = kk;
            stk[2 * sp + 2] = kk + 1; stk[2 * sp + 3] = j;
          }
          sp += 2;
        }
      }
      if (lane == 0) {
        status[b] = badsh ? SDB_ST_INVALID : SDB_ST_OK;
        score[b] = Z;
      }
    }
    return;
  }

  // ---- 3. outside (constituency.py:84-99)
  for (int e = tid; e < (int)T; e += kThreads) out[e] = ninfd();
  __syncthreads();
  if (tid == 0) out[tri(0, n - 1, n)] = 0.0;
  __syncthreads();
  for (int w = n - 1; w >= 1; --w) {
    const int nterms = n - w;
    for (int i = warp; i <= n - w; i += kWarps) {
      const int j = i + w - 1;
      const int nr = n - 1 - j;  // right-sibling parents (i, pj), pj in (j, n)
      // each lane holds <= 4 parent terms (n <= 128): read them once
      double tv[4];
      double mloc = ninfd();
#pragma unroll
      for (int r4 = 0; r4 < 4; ++r4) {
        const int q = lane + 32 * r4;
        double t = ninfd();
        if (q < nterms) {
          if (q < nr) {
            const int pj = j + 1 + q;
            t = out[tri(i, pj, n)] + (double)fold[tri(i, pj, n)] + ins[tri(j + 1, pj, n)];
          } else {
            const int pi = q - nr;
            t = out[tri(pi, j, n)] + (double)fold[tri(pi, j, n)] + ins[tri(pi, i - 1, n)];
          }
        }
        tv[r4] = t;
        mloc = fmax(mloc, t);
      }
      float s = 0.f;
      if (mloc != ninfd())
#pragma unroll
        for (int r4 = 0; r4 < 4; ++r4) s += (tv[r4] == ninfd()) ? 0.f : fexp((float)(tv[r4] - mloc));
      const double r = warp_lse_d(mloc, s);
      if (lane == 0) out[tri(i, j, n)] = r;
    }
    __syncthreads();
  }

  // ---- 4. marginals over the full [n][n][m] output
  float* mg = marg_all + (size_t)b * n * n * m;
  const bool vec = (m & 3) == 0;
  const int mq = vec ? m / 4 : m;
  const size_t tot = (size_t)n * n * mq;
  for (size_t e = tid; e < tot; e += kThreads) {
    const int ij = (int)(e / mq), q = (int)(e - (size_t)ij * mq);
    const int i = ij / n, j = ij - i * n;
    float K = 0.f;
    bool live = false;
    if (i <= j) {
      const int t = tri(i, j, n);
      const double o = out[t], in = ins[t];
      if (o != ninfd() && in != ninfd()) {
        live = true;
        K = (float)(o + in - (double)fold[t] - Z);
      }
    }
    if (vec) {
      float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
      if (live) {
        const float4 x = *reinterpret_cast<const float4*>(th + (size_t)ij * m + 4 * q);
        r.x = fexp(K + x.x); r.y = fexp(K + x.y); r.z = fexp(K + x.z); r.w = fexp(K + x.w);
      }
      reinterpret_cast<float4*>(mg)[e] = r;
    } else {
      mg[e] = live ? fexp(K + th[(size_t)ij * m + q]) : 0.f;
    }
  }
  if (tid == 0) {
    status[b] = badsh ? SDB_ST_INVALID : SDB_ST_OK;
    logz[b] = Z;
  }
}

template <int kMode>
int tree_launch(const float* th, int64_t B, int n, int m, double* logz, float* marg, int32_t* labels, double* score,
                int32_t* status, cudaStream_t s) {
  const size_t smem = tree_smem(n);
  if (cudaFuncSetAttribute(tree_kernel<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SDB_ERR_CUDA;
  tree_kernel<kMode><<<(unsigned)B, kThreads, smem, s>>>(th, n, m, logz, marg, labels, score, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

int tree_check(int64_t B, int n, int m) {
  if (B < 0 || n < 1 || m < 1) return SDB_ERR_ARG;
  if (n > 128 || tree_smem(n) > 220 * 1024) return SDB_ERR_UNSUPPORTED;  // <= 4 terms per lane
  return SDB_OK;
}

}  // namespace

extern "C" int sdb_tree_fb(const float* span_potentials, int64_t B, int32_t n, int32_t m, double* logz, float* marg,
                           int32_t* status, void* stream) {
  int rc = tree_check(B, n, m);
  if (rc) return rc;
  if (!span_potentials || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (marg) return tree_launch<1>(span_potentials, B, n, m, logz, marg, nullptr, nullptr, status, s);
  return tree_launch<0>(span_potentials, B, n, m, logz, nullptr, nullptr, nullptr, status, s);
}

extern "C" int sdb_tree_viterbi(const float* span_potentials, int64_t B, int32_t n, int32_t m, int32_t* labels,
                                double* score, int32_t* status, void* stream) {
  int rc = tree_check(B, n, m);
  if (rc) return rc;
  if (!span_potentials || !labels || !score || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  return tree_launch<2>(span_potentials, B, n, m, nullptr, nullptr, labels, score, status, (cudaStream_t)stream);
}
