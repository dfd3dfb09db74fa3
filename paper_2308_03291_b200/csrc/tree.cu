// Span-factored Tree-CRF (CKY): log-partition, labeled-span marginals,
// max-plus argmax.
//
// Reference: structdist constituency.py:52-133 (_tree_charts,
// cky_log_partition, tree_marginals, _tree_walk, tree_argmax).
// Layout per instance: span_potentials [n][n][m] fp32 (only i <= j is read;
// marginals for i > j are written as 0).
//
// log_partition + marginals (sdb_tree_fb) is a chain of three kernels, see
// the block comment above tree_fold_kernel: label fold (HBM) -> scaled-linear
// inside/outside (one CTA per instance, latency-bound) -> marginal emission
// (HBM).  tree_kernel below is the exact log-space path: the max-plus argmax
// (kMode 2) and the fallback for instances the linear charts cannot hold:
//   1. label fold: fold[i,j] = lse_l theta[i,j,l] (thread per span);
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
constexpr int32_t kRetry = 5;  // scaled-linear DP could not represent this instance

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
                                                         double* __restrict__ score, int32_t* __restrict__ status,
                                                         int only_retry) {
  // fallback use: redo only the instances the scaled-linear path gave up on
  if (only_retry && status[blockIdx.x] != kRetry) return;
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

// ===========================================================================
// Scaled-linear path for log_partition + marginals (the C5a hot path).
//
//   tree_fold_kernel  (HBM):     fold[b][i,j] = lse_l theta[b,i,j,l], a warp per
//                                (b, i) row: the spans j = i..n-1 of one row are
//                                contiguous, so the row streams with coalesced
//                                16-byte loads, m/4 lanes per span.
//   tree_lin_kernel   (latency): one CTA per instance; inside and outside over
//                                F = exp(fold) 2^-e in LINEAR fp32 (every tree
//                                over a width-w span has 2w-1 nodes, so the
//                                per-node factor 2^-e scales each width
//                                uniformly and cancels exactly in
//                                outside*inside/Z); split sums are dot products
//                                of two contiguous chart rows/columns (packed
//                                row-major and column-major copies).  Writes
//                                K[i,j] = log(O I / Z) - fold[i,j] per span.
//   tree_emit_kernel  (HBM):     marg[b,i,j,l] = exp(K[i,j] + theta[b,i,j,l]),
//                                zeros for i > j; a CTA per (b, i) row.
// Instances whose linear charts leave [2^-110, 2^110] (or hold a -inf fold)
// are flagged kRetry and recomputed by the log-space tree_kernel.
// ===========================================================================

constexpr int kFoldWarps = 8;

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
constexpr int kEmitThreads = 256;
constexpr float kLinHi = 1.2980742e33f;   // 2^110
constexpr float kLinLo = 7.7037198e-34f;  // 2^-110

// lse over one label row held as QV float4 in registers (QV compile-time: no
// register array sized for the largest m, so the occupancy stays high)
template <int QV>
__device__ __forceinline__ float fold_row(const float4* __restrict__ r4) {
  float4 v[QV];
#pragma unroll
  for (int u = 0; u < QV; ++u) v[u] = __ldg(r4 + u);
  // NaN-propagating max: NaN or +inf anywhere in the row -> !(mx < +inf)
  float mx = ninf();
#pragma unroll
  for (int u = 0; u < QV; ++u) mx = fmax_nan(mx, fmax_nan(fmax_nan(v[u].x, v[u].y), fmax_nan(v[u].z, v[u].w)));
  const int bad = !(mx < __int_as_float(0x7f800000));
  float s = 0.f;
  if (!bad && mx != ninf()) {
#pragma unroll
    for (int u = 0; u < QV; ++u) s += (fexp(v[u].x - mx) + fexp(v[u].y - mx)) + (fexp(v[u].z - mx) + fexp(v[u].w - mx));
  }
  return bad ? __int_as_float(0x7fc00000) : ((mx == ninf()) ? ninf() : mx + flog(s));
}

// QV = m/4 when m is 16, 32 or 64 (16-byte rows), 0 = generic scalar path
template <int QV>
__global__ void __launch_bounds__(kFoldWarps * 32) tree_fold_kernel(const float* __restrict__ th_all, int64_t B,
                                                                    int n, int m, float* __restrict__ fold_all) {
  const int64_t row = (int64_t)blockIdx.x * kFoldWarps + (threadIdx.x >> 5);
  if (row >= B * n) return;
  const int lane = threadIdx.x & 31;
  const int64_t b = row / n;
  const int i = (int)(row - b * n);
  const int T = n * (n + 1) / 2;
  const float* src = th_all + ((size_t)row * n + i) * m;  // theta[b, i, i, 0]
  float* dst = fold_all + (size_t)b * T + tri(i, i, n);
  const int ns = n - i;
  if (QV > 0) {
    // lane per span: the lane's label row is m/4 16-byte loads, all issued
    // before the (max, sum) pass; a warp-instruction touches 32 rows but every
    // fetched sector is consumed
    for (int sp = lane; sp < ns; sp += 32)
      dst[sp] = fold_row<(QV > 0 ? QV : 1)>(reinterpret_cast<const float4*>(src + (size_t)sp * m));
  } else {
    for (int sp = lane; sp < ns; sp += 32) {
      const float* rw = src + (size_t)sp * m;
      Lse acc;
      int bad = 0;
      for (int l = 0; l < m; ++l) {
        const float x = __ldg(rw + l);
        bad |= bad_input(x);
        acc.add(x);
      }
      dst[sp] = bad ? __int_as_float(0x7fc00000) : acc.result();
    }
  }
}


// Charts: packed row-major (R: chart[i, i..n-1] at rs(i)) and packed
// column-major (C: chart[0..j, j] at cs(j)) copies, so the split terms of a
// span are contiguous in both operands.  A span of width w gets G = 2^LG lanes
// (<= 8 terms per lane); lane r takes terms r, r+G, ..., so for a fixed term
// the G lanes of a span read G consecutive words.  The step body is
// instantiated per LG: term offsets are immediates, loads are predicated (no
// branches), and a step costs ~50 instructions per warp.
constexpr int kLinThreads = 512;

__device__ __forceinline__ int rs(int i, int n) { return i * n - ((i * (i - 1)) >> 1); }  // == tri(i, i, n)
__device__ __forceinline__ int cs(int j) { return (j * (j + 1)) >> 1; }

struct LinCharts {
  float *base, *fl, *Fr, *Ir, *Ic, *Pr, *Pc;
  int zi;  // index of a shared zero word (masked operands read it)
};

template <int LG>
__device__ __forceinline__ int inside_step(const LinCharts& c, int n, int w, int tid, int bad) {
  constexpr int G = 1 << LG;
  const int L = w - 1, nsp = n - w + 1, r = tid & (G - 1);
  const int wfirst = (tid & ~31) >> LG;
  for (int base = 0; base < nsp; base += kLinThreads >> LG) {
    if (base + wfirst >= nsp) break;  // warp-uniform
    const int i = base + (tid >> LG), j = i + w - 1;
    const bool ok = i < nsp;
    // operand indices relative to c.base; masked terms read the zero slot (no branches)
    const int p = (int)(c.Ir - c.base) + rs(i, n) + r;  // I[i, i + t]
    const int q = (int)(c.Ic - c.base) + cs(j) + i + 1 + r;  // I[i + 1 + t, j]
    const int lim = ok ? L - r : 0;
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool pr = u * G < lim;
      const float x = c.base[pr ? p + u * G : c.zi], y = c.base[pr ? q + u * G : c.zi];
      if (u & 1) a1 = fmaf(x, y, a1); else a0 = fmaf(x, y, a0);
    }
    float acc = a0 + a1;
#pragma unroll
    for (int o = G >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (ok && r == 0) {
      const int t = rs(i, n) + w - 1;
      const float v = acc * c.Fr[t];
      bad |= !(v >= kLinLo && v <= kLinHi);
      c.Ir[t] = v;
      c.Ic[cs(j) + i] = v;
    }
  }
  return bad;
}

template <int LG>
__device__ __forceinline__ int outside_step(const LinCharts& c, int n, int w, int tid, int bad, float lz2,
                                            float* __restrict__ Kb) {
  constexpr int G = 1 << LG;
  const int L = n - w, nsp = n - w + 1, r = tid & (G - 1);
  const int wfirst = (tid & ~31) >> LG;
  for (int base = 0; base < nsp; base += kLinThreads >> LG) {
    if (base + wfirst >= nsp) break;  // warp-uniform
    const int i = base + (tid >> LG), j = i + w - 1, nr = n - 1 - j;
    const bool ok = i < nsp;
    // right-sibling parents (i, j+1+t), t < nr: P[i, j+1+t] (row i), I[j+1, j+1+t] (row j+1)
    const int pa = (int)(c.Pr - c.base) + rs(i, n) + w + r;
    const int pb = (int)(c.Ir - c.base) + rs(j + 1, n) + r;
    // left-sibling parents (t - nr, j), t >= nr: P[t-nr, j] (column j), I[t-nr, i-1] (column i-1)
    const int qa = (int)(c.Pc - c.base) + cs(j) - nr + r;
    const int qb = (int)(c.Ic - c.base) + cs(i - 1) - nr + r;
    const int lim = ok ? L - r : 0, rlim = nr - r;
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool pr = u * G < lim, right = u * G < rlim;
      const int xa = pr ? (right ? pa : qa) + u * G : c.zi;
      const int xb = pr ? (right ? pb : qb) + u * G : c.zi;
      const float x = c.base[xa], y = c.base[xb];
      if (u & 1) a1 = fmaf(x, y, a1); else a0 = fmaf(x, y, a0);
    }
    float acc = a0 + a1;
#pragma unroll
    for (int o = G >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (ok && r == 0) {
      const int t = rs(i, n) + w - 1;
      bad |= !(acc >= kLinLo && acc <= kLinHi);
      const float pv = acc * c.Fr[t];
      c.Pr[t] = pv;
      c.Pc[cs(j) + i] = pv;
      Kb[t] = (lg2(acc) + lg2(c.Ir[t]) - lz2) * SDB_LN2 - c.fl[t];
    }
  }
  return bad;
}

template <bool kMarg>
__global__ void __launch_bounds__(kLinThreads) tree_lin_kernel(const float* __restrict__ fold_all, int n,
                                                              double* __restrict__ logz, float* __restrict__ K_all,
                                                              int32_t* __restrict__ status) {
  extern __shared__ __align__(16) float sml[];
  const int T = n * (n + 1) / 2;
  LinCharts c;
  c.base = sml;
  c.zi = 6 * T;
  c.fl = sml;         // fold (log), row-major
  c.Fr = c.fl + T;    // F' = exp(fold) 2^-e, row-major
  c.Ir = c.Fr + T;    // inside, row-major
  c.Ic = c.Ir + T;    // inside, column-major
  c.Pr = c.Ic + T;    // outside * F', row-major
  c.Pc = c.Pr + T;    // outside * F', column-major
  __shared__ float red[2][kLinThreads / 32];
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- load fold; NaN -> invalid, -inf -> retry (the log-space kernel handles
  // -inf structure exactly)
  const float* fsrc = fold_all + (size_t)b * T;
  float mx = ninf();
  int flg = 0;
  if (tid == 0) sml[c.zi] = 0.f;
  for (int t0 = 0; t0 < T; t0 += kLinThreads * 4) {
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = t0 + kLinThreads * u + tid;
      v[u] = (t < T) ? fsrc[t] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = t0 + kLinThreads * u + tid;
      if (t < T) {
        const float f = v[u];
        c.fl[t] = f;
        if (f != f) flg |= 1;
        else if (f == ninf()) flg |= 2;
        else mx = fmaxf(mx, f);
      }
    }
  }
  mx = warp_max(mx);
  if (lane == 0) red[0][warp] = mx;
  flg = (__syncthreads_or(flg & 1) ? 1 : 0) | (__syncthreads_or(flg & 2) ? 2 : 0);
  if (flg) {
    if (tid == 0) {
      status[b] = (flg & 1) ? SDB_ST_INVALID : kRetry;
      logz[b] = (flg & 1) ? __longlong_as_double(0x7ff8000000000000ULL) : ninfd();
    }
    return;
  }
  mx = red[0][0];
#pragma unroll
  for (int k = 1; k < kLinThreads / 32; ++k) mx = fmaxf(mx, red[0][k]);
  float s = 0.f;
  for (int t = tid; t < T; t += kLinThreads) s += fexp(c.fl[t] - mx);
  s = warp_sum(s);
  if (lane == 0) red[1][warp] = s;
  __syncthreads();
  float st = 0.f;
#pragma unroll
  for (int k = 0; k < kLinThreads / 32; ++k) st += red[1][k];
  // per-node scale: twice the mean factor (Catalan growth ~4^w over 2w-1 nodes)
  const float e = mx * SDB_LOG2E + lg2(st / (float)T) + 1.f;
  int bad = 0;
  for (int t = tid; t < T; t += kLinThreads) {
    const float f = ex2(fmaf(c.fl[t], SDB_LOG2E, -e));
    bad |= !(f >= kLinLo && f <= kLinHi);
    c.Fr[t] = f;
  }
  __syncthreads();
  for (int i = tid; i < n; i += kLinThreads) {
    const float f = c.Fr[rs(i, n)];
    c.Ir[rs(i, n)] = f;
    c.Ic[cs(i) + i] = f;
  }
  // ---- inside (constituency.py:57-63): I[i,j] = F'[i,j] sum_k I[i,k] I[k+1,j]
  // widths with the same lane-group size are contiguous (L = w-1 <= 8 * 2^LG): one
  // specialised loop per group size instead of a per-width indirect branch
  for (int w = 2; w <= min(n, 9); ++w) { __syncthreads(); bad = inside_step<0>(c, n, w, tid, bad); }
  for (int w = 10; w <= min(n, 17); ++w) { __syncthreads(); bad = inside_step<1>(c, n, w, tid, bad); }
  for (int w = 18; w <= min(n, 33); ++w) { __syncthreads(); bad = inside_step<2>(c, n, w, tid, bad); }
  for (int w = 34; w <= min(n, 65); ++w) { __syncthreads(); bad = inside_step<3>(c, n, w, tid, bad); }
  for (int w = 66; w <= n; ++w) { __syncthreads(); bad = inside_step<4>(c, n, w, tid, bad); }
  bad = __syncthreads_or(bad);
  const float Zs = c.Ir[rs(0, n) + n - 1];
  if (bad) {
    if (tid == 0) status[b] = kRetry;
    return;
  }
  if (tid == 0) logz[b] = log((double)Zs) + (double)e * (double)(2 * n - 1) * 0.6931471805599453;
  if (!kMarg) {
    if (tid == 0) status[b] = SDB_ST_OK;
    return;
  }
  // ---- outside (constituency.py:84-99) over P = O' F'; K = log(O' I' / Z') - fold
  float* Kb = K_all + (size_t)b * T;  // row-major packed (read by tree_emit_kernel)
  const float lz2 = lg2(Zs);
  if (tid == 0) {
    const int t = n - 1;  // root (0, n-1)
    c.Pr[t] = c.Fr[t];
    c.Pc[cs(n - 1)] = c.Fr[t];
    Kb[t] = -c.fl[t];  // O' I' / Z' = 1 at the root
  }
  // L = n - w grows as w falls: the same contiguous group-size ranges, in reverse
  for (int w = n - 1; w >= max(1, n - 8); --w) { __syncthreads(); bad = outside_step<0>(c, n, w, tid, bad, lz2, Kb); }
  for (int w = n - 9; w >= max(1, n - 16); --w) { __syncthreads(); bad = outside_step<1>(c, n, w, tid, bad, lz2, Kb); }
  for (int w = n - 17; w >= max(1, n - 32); --w) { __syncthreads(); bad = outside_step<2>(c, n, w, tid, bad, lz2, Kb); }
  for (int w = n - 33; w >= max(1, n - 64); --w) { __syncthreads(); bad = outside_step<3>(c, n, w, tid, bad, lz2, Kb); }
  for (int w = n - 65; w >= 1; --w) { __syncthreads(); bad = outside_step<4>(c, n, w, tid, bad, lz2, Kb); }
  bad = __syncthreads_or(bad);
  if (tid == 0) status[b] = bad ? kRetry : SDB_ST_OK;
}

__global__ void __launch_bounds__(kEmitThreads) tree_emit_kernel(const float* __restrict__ th_all, int n, int m,
                                                                 int qshift, const float* __restrict__ K_all,
                                                                 const int32_t* __restrict__ status,
                                                                 float* __restrict__ marg_all) {
  const int64_t row = blockIdx.x;
  const int64_t b = row / n;
  const int i = (int)(row - b * n);
  const int st = status[b];
  if (st == kRetry) return;  // the log-space kernel writes this instance
  const bool live = st == SDB_ST_OK;
  const int T = n * (n + 1) / 2;
  const float* Kr = K_all + (size_t)b * T + tri(i, i, n) - i;  // Kr[j] = K[i, j] for j >= i
  const float* src = th_all + (size_t)row * n * m;
  float* dst = marg_all + (size_t)row * n * m;
  if (qshift >= 0) {
    const int tot = n << qshift;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    // two float4 per thread per pass, both loads issued before the stores
    for (int x0 = threadIdx.x; x0 < tot; x0 += 2 * kEmitThreads) {
      const int x1 = x0 + kEmitThreads;
      const int j0 = x0 >> qshift, j1 = x1 >> qshift;
      const bool l0 = live && j0 >= i, l1 = live && x1 < tot && j1 >= i;
      float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
      float k0 = 0.f, k1 = 0.f;
      if (l0) { v0 = __ldg(s4 + x0); k0 = Kr[j0]; }
      if (l1) { v1 = __ldg(s4 + x1); k1 = Kr[j1]; }
      float4 o0 = make_float4(0.f, 0.f, 0.f, 0.f), o1 = o0;
      if (l0) { o0.x = fexp(k0 + v0.x); o0.y = fexp(k0 + v0.y); o0.z = fexp(k0 + v0.z); o0.w = fexp(k0 + v0.w); }
      if (l1) { o1.x = fexp(k1 + v1.x); o1.y = fexp(k1 + v1.y); o1.z = fexp(k1 + v1.z); o1.w = fexp(k1 + v1.w); }
      d4[x0] = o0;
      if (x1 < tot) d4[x1] = o1;
    }
  } else {
    const int tot = n * m;
    for (int x = threadIdx.x; x < tot; x += kEmitThreads) {
      const int j = x / m;
      dst[x] = (live && j >= i) ? fexp(Kr[j] + __ldg(src + x)) : 0.f;
    }
  }
}

size_t tree_ws(int64_t B, int n) {
  Carve c(nullptr);
  const size_t T = (size_t)n * (n + 1) / 2;
  c.take<float>((size_t)B * T);
  c.take<float>((size_t)B * T);
  return c.used;
}

template <int kMode>
int tree_launch(const float* th, int64_t B, int n, int m, double* logz, float* marg, int32_t* labels, double* score,
                int32_t* status, cudaStream_t s, int only_retry = 0) {
  const size_t smem = tree_smem(n);
  if (sdb_set_smem((const void*)tree_kernel<kMode>, smem) != cudaSuccess)
    return SDB_ERR_CUDA;
  tree_kernel<kMode><<<(unsigned)B, kThreads, smem, s>>>(th, n, m, logz, marg, labels, score, status, only_retry);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

bool tree_fast_ok(int n) { return n <= 128 && tree_smem(n) <= 220 * 1024; }  // <= 4 terms per lane

}  // namespace

// tree_gen.cu: fp64 charts in global memory for longer sentences
bool tree_gen_ok(int n);
size_t tree_gen_workspace(int64_t B, int n);
int tree_gen_launch(int mode, const float* sp, int64_t B, int n, int m, void* ws, size_t ws_bytes, double* out,
                    float* marg, int32_t* labels, int32_t* status, cudaStream_t s);

namespace {
int tree_check(int64_t B, int n, int m) {
  if (B < 0 || n < 1 || m < 1) return SDB_ERR_ARG;
  if (!tree_fast_ok(n) && !tree_gen_ok(n)) return SDB_ERR_UNSUPPORTED;
  return SDB_OK;
}
}  // namespace

extern "C" size_t sdb_tree_fb_workspace(int64_t B, int32_t n, int32_t m) {
  (void)m;
  if (B > 0 && n > 0 && !tree_fast_ok(n)) return tree_gen_workspace(B, n);
  return (B > 0 && n > 0) ? tree_ws(B, n) : 0;
}

extern "C" int sdb_tree_fb(const float* span_potentials, int64_t B, int32_t n, int32_t m, double* logz, float* marg,
                           int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  int rc = tree_check(B, n, m);
  if (rc) return rc;
  if (!span_potentials || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!tree_fast_ok(n)) {
    if (!workspace) return SDB_ERR_WORKSPACE;
    return tree_gen_launch(marg ? 1 : 0, span_potentials, B, n, m, workspace, ws_bytes, logz, marg, nullptr, status,
                           (cudaStream_t)stream);
  }
  if (!workspace || ws_bytes < tree_ws(B, n)) return SDB_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  Carve c(workspace);
  const size_t T = (size_t)n * (n + 1) / 2;
  float* fold = c.take<float>((size_t)B * T);
  float* K = c.take<float>((size_t)B * T);
  const size_t smem_lin = (6 * T + 1) * sizeof(float);
  if (sdb_set_smem((const void*)tree_lin_kernel<true>, smem_lin) !=
          cudaSuccess ||
      sdb_set_smem((const void*)tree_lin_kernel<false>, smem_lin) !=
          cudaSuccess)
    return SDB_ERR_CUDA;
  const int64_t rows = B * n;
  {
    const unsigned fg = (unsigned)((rows + kFoldWarps - 1) / kFoldWarps);
    const bool al16 = (((uintptr_t)span_potentials) & 15) == 0;
    if (al16 && m == 32) tree_fold_kernel<8><<<fg, kFoldWarps * 32, 0, s>>>(span_potentials, B, n, m, fold);
    else if (al16 && m == 16) tree_fold_kernel<4><<<fg, kFoldWarps * 32, 0, s>>>(span_potentials, B, n, m, fold);
    else if (al16 && m == 64) tree_fold_kernel<16><<<fg, kFoldWarps * 32, 0, s>>>(span_potentials, B, n, m, fold);
    else tree_fold_kernel<0><<<fg, kFoldWarps * 32, 0, s>>>(span_potentials, B, n, m, fold);
  }
  SDB_CHECK_LAUNCH();
  if (marg) {
    tree_lin_kernel<true><<<(unsigned)B, kLinThreads, smem_lin, s>>>(fold, n, logz, K, status);
    SDB_CHECK_LAUNCH();
    int qshift = -1;
    if ((m & 3) == 0 && (((uintptr_t)span_potentials | (uintptr_t)marg) & 15) == 0) {
      const int q = m >> 2;
      if ((q & (q - 1)) == 0) qshift = __builtin_ctz(q);
    }
    tree_emit_kernel<<<(unsigned)rows, kEmitThreads, 0, s>>>(span_potentials, n, m, qshift, K, status, marg);
    SDB_CHECK_LAUNCH();
    return tree_launch<1>(span_potentials, B, n, m, logz, marg, nullptr, nullptr, status, s, 1);
  }
  tree_lin_kernel<false><<<(unsigned)B, kLinThreads, smem_lin, s>>>(fold, n, logz, K, status);
  SDB_CHECK_LAUNCH();
  return tree_launch<0>(span_potentials, B, n, m, logz, nullptr, nullptr, nullptr, status, s, 1);
}

extern "C" int sdb_tree_viterbi(const float* span_potentials, int64_t B, int32_t n, int32_t m, int32_t* labels,
                                double* score, int32_t* status, void* stream) {
  int rc = tree_check(B, n, m);
  if (rc) return rc;
  if (!span_potentials || !labels || !score || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!tree_fast_ok(n))
    return tree_gen_launch(2, span_potentials, B, n, m, nullptr, 0, score, nullptr, labels, status,
                           (cudaStream_t)stream);
  return tree_launch<2>(span_potentials, B, n, m, nullptr, nullptr, labels, score, status, (cudaStream_t)stream);
}
