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
// For m <= 32 (the C1 shape) log_partition + marginals take the scaled-LINEAR
// path instead (chain_lin_kernel + chain_lin_marg_kernel below); this
// log-space path serves larger m and the instances the linear path flags.
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
  int32_t* need;  // [B] 1 = recompute with the exact log-space path
  int32_t* needb; // [B] linear backward pass verdict (merged into `need` by the emission kernel)
};

__host__ ChainWs carve_chain(void* base, int64_t B, int n, int m, size_t* bytes) {
  Carve c(base);
  ChainWs w;
  w.alpha = c.take<float>((size_t)B * n * m);
  w.beta = c.take<float>((size_t)B * n * m);
  w.acum = c.take<double>((size_t)B * n);
  w.bcum = c.take<double>((size_t)B * n);
  w.flags = c.take<int32_t>((size_t)B);
  w.need = c.take<int32_t>((size_t)B);
  w.needb = c.take<int32_t>((size_t)B);
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

// ---------------------------------------------------------------------
// Fast path for m <= 32 (the C1 shape): every step's m x m potentials are
// prefetched kD steps ahead into a shared ring with cp.async (16-byte chunks
// when the step is 16-byte aligned); the 8 warps split the rows (forward) or
// rows-by-warp (backward) and warp 0 finishes the step with warp-level
// reductions, so a step costs two CTA barriers and no global-load latency.
constexpr int kD = 8;

__device__ __forceinline__ void cpa16(float* dst, const float* src) {
  unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cpa4(float* dst, const float* src) {
  unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cpa_wait_d() { asm volatile("cp.async.wait_group %0;\n" ::"n"(kD - 1)); }

__device__ __forceinline__ void stage_step(float* dst, const float* src, int mm, bool v16) {
  if (v16) {
    for (int e = threadIdx.x; e < (mm >> 2); e += kThreads) cpa16(dst + 4 * e, src + 4 * e);
  } else {
    for (int e = threadIdx.x; e < mm; e += kThreads) cpa4(dst + e, src + e);
  }
}

__global__ void __launch_bounds__(kThreads) chain_fwd_bwd_small_kernel(
    const float* __restrict__ init, const float* __restrict__ trans, int n, int m, ChainWs ws,
    double* __restrict__ logz, int32_t* __restrict__ status, int only_need) {
  if (only_need && ws.need[blockIdx.x] == 0) return;
  extern __shared__ __align__(16) float sm[];
  const int mm = m * m;
  float* stage = sm;                     // [kD][mm]
  float* vec = stage + kD * mm;          // [32]
  float* pm = vec + 32;                  // [kGroups][32]
  float* ps = pm + kGroups * 32;         // [kGroups][32]
  __shared__ int redi[kThreads / 32];
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* th = trans + (size_t)b * (n - 1) * mm;
  const bool v16 = ((mm & 3) == 0);
  const bool fwd = blockIdx.y == 0;
  int bad = 0;
  // prologue prefetch: steps in processing order
  for (int d = 0; d < kD; ++d) {
    const int t = fwd ? d : n - 2 - d;
    if (d < n - 1) stage_step(stage + d * mm, th + (size_t)t * mm, mm, v16);
    cpa_commit();
  }
  if (fwd) {
    float* al = ws.alpha + (size_t)b * n * m;
    double* ac = ws.acum + (size_t)b * n;
    double A = 0.0;
    bool vac = false;
    if (warp == 0) {
      const float x = lane < m ? init[(size_t)b * m + lane] : ninf();
      bad |= (lane < m) && bad_input(x);
      float c = warp_max(x);
      vac = (c == ninf());
      A = vac ? 0.0 : (double)c;
      if (vac) c = 0.f;
      if (lane < m) {
        vec[lane] = x - c;
        al[lane] = x - c;
      }
      if (lane == 0) ac[0] = A;
    }
    for (int t = 0; t < n - 1; ++t) {
      cpa_wait_d();
      __syncthreads();  // step t resident; vec of step t visible
      const float* tt = stage + (t % kD) * mm;
      if (lane < m) {
        Lse acc;
        for (int a = warp; a < m; a += kGroups) {
          const float x = tt[a * m + lane];
          bad |= bad_input(x);
          acc.add(vec[a] + x);
        }
        pm[warp * 32 + lane] = acc.m;
        ps[warp * 32 + lane] = acc.s;
      }
      __syncthreads();  // partials visible; everybody is done reading slot t % kD and vec
      {
        const int tn = t + kD;
        if (tn < n - 1) stage_step(stage + (t % kD) * mm, th + (size_t)tn * mm, mm, v16);
        cpa_commit();
      }
      if (warp == 0) {
        Lse acc;
        if (lane < m) {
#pragma unroll
          for (int g = 0; g < kGroups; ++g) acc.merge(pm[g * 32 + lane], ps[g * 32 + lane]);
        }
        const float u = lane < m ? acc.result() : ninf();
        float c = warp_max(u);
        if (c == ninf()) vac = true;
        if (vac) c = 0.f;
        A += (double)c;
        if (lane < m) {
          const float v = vac ? ninf() : u - c;
          vec[lane] = v;
          al[(size_t)(t + 1) * m + lane] = v;
        }
        if (lane == 0) ac[t + 1] = A;
      }
    }
    bad = block_or(bad, redi);
    if (warp == 0) {
      float z = ninf();
      if (!vac) {
        const float v = lane < m ? vec[lane] : ninf();
        z = warp_lse(v);
      }
      if (lane == 0) {
        vac = vac || z == ninf();
        logz[b] = vac ? ninfd() : A + (double)z;
        const int st = bad ? SDB_ST_INVALID : (vac ? SDB_ST_VACUOUS : SDB_ST_OK);
        status[b] = st;
        ws.flags[b] = st;
      }
    }
  } else {
    float* be = ws.beta + (size_t)b * n * m;
    double* bc = ws.bcum + (size_t)b * n;
    double Bc = 0.0;
    if (warp == 0 && lane < m) {
      vec[lane] = 0.f;
      be[(size_t)(n - 1) * m + lane] = 0.f;
    }
    if (tid == 0) bc[n - 1] = 0.0;
    for (int d = 0; d < n - 1; ++d) {
      const int t = n - 2 - d;
      cpa_wait_d();
      __syncthreads();
      const float* tt = stage + (d % kD) * mm;
      const float bv = lane < m ? vec[lane] : ninf();
      for (int a = warp; a < m; a += kGroups) {
        const float x = lane < m ? tt[a * m + lane] + bv : ninf();
        const float r = warp_lse(x);
        if (lane == 0) pm[a] = r;
      }
      __syncthreads();
      {
        const int dn = d + kD;
        if (dn < n - 1) stage_step(stage + (d % kD) * mm, th + (size_t)(n - 2 - dn) * mm, mm, v16);
        cpa_commit();
      }
      if (warp == 0) {
        const float r = lane < m ? pm[lane] : ninf();
        float dd = warp_max(r);
        if (dd == ninf()) dd = 0.f;
        Bc += (double)dd;
        if (lane < m) {
          vec[lane] = r - dd;
          be[(size_t)t * m + lane] = r - dd;
        }
        if (lane == 0) bc[t] = Bc;
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
}

// ---------------------------------------------------------------------
// Linear-space kernel for m <= 32 (the C1 shape).
//
// Two CTAs per instance, independent: blockIdx.x & 1 == 0 runs the forward
// recurrence, 1 the backward one, concurrently.  Inside a CTA:
//   * warp 0 runs the recurrence in scaled LINEAR space: a step is a 32x32
//     mat-vec of FMAs, u_x = sum_y M_t[x][y] v_y (lane x reads its row and the
//     broadcast vector as float4), renormalised by its max (one REDUX + one
//     MUFU.RCP), with the log scale accumulated in fp64 -- no exp/log on the
//     critical path; every vector and its scale go to the workspace;
//   * warps 1-7 are producers: they cp.async-stage the raw potentials two
//     7-step blocks ahead and convert them to E_t = exp(theta_t) one block
//     ahead (a zero / non-finite state in the recurrence flags the instance
//     for the exact log-space fallback).
// The marginals are NOT emitted here (they used to be, by the producers after
// a meet-in-the-middle exchange, which made the producers the bottleneck):
// chain_lin_marg_kernel streams them from the stored vectors with a grid over
// (step block, instance), so this kernel's time is the recurrence itself.
// E rings are stored output-major (forward: E^T, backward: E) with a 36-float
// pitch so the recurrence reads rows as float4.
constexpr int kLB = kGroups - 1;        // steps per block = producer warps (one step each)
constexpr int kEP = 36;                // padded row pitch (16-byte aligned rows for LDS.128)
constexpr int kERing = 3 * kLB;        // E slots: blocks k-1 (emit), k (consume), k+1 (produce)
constexpr int kRRing = 3 * kLB;        // raw slots: blocks k+1, k+2, k+3

struct LinSmem {
  float* raw;      // [kRRing][1024]
  float* E;        // [kERing][32][kEP]
  float* Mt;       // [kERing] step max (natural log)
  uint32_t* mask;  // [kERing][32] finiteness masks (fwd: per column b bits over a; bwd: per row a bits over b)
};

size_t lin_smem_bytes() {
  return (size_t)kRRing * 1024 * 4 + (size_t)kERing * 32 * kEP * 4 + kERing * 4 + kERing * 32 * 4 + 256;
}

__global__ void __launch_bounds__(kThreads, 1)
    chain_lin_kernel(const float* __restrict__ init, const float* __restrict__ trans, int n, int m, ChainWs ws,
                     double* __restrict__ logz, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) char smraw[];
  LinSmem S;
  {
    char* p = smraw;
    S.raw = (float*)p; p += (size_t)kRRing * 1024 * 4;
    S.E = (float*)p; p += (size_t)kERing * 32 * kEP * 4;
    S.mask = (uint32_t*)p; p += (size_t)kERing * 32 * 4;
    S.Mt = (float*)p;
  }
  __shared__ int flagsh;  // bit0 invalid input, bit1 fallback needed
  __shared__ __align__(16) float vsh[32];
  const int dir = blockIdx.x & 1;  // 0 forward, 1 backward
  const int b = blockIdx.x >> 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = n - 1;
  const int mm = m * m;
  const float* th = trans + (size_t)b * T * mm;
  float* vecs = dir == 0 ? ws.alpha + (size_t)b * n * m : ws.beta + (size_t)b * n * m;   // linear e_t / f_t
  double* scs = dir == 0 ? ws.acum + (size_t)b * n : ws.bcum + (size_t)b * n;         // their log scales
  const int NB = (T + kLB - 1) / kLB;
  if (tid == 0) flagsh = 0;
  // step index of processing position q
  auto tstep = [&](int q) { return dir == 0 ? q : T - 1 - q; };
  const bool v16 = ((mm & 3) == 0);
  auto issue_raw = [&](int blk) {  // producer warp w-1 stages step w-1 of block blk (own cp.async group)
    const int q = blk * kLB + (warp - 1);
    if (blk < NB && q < T) {
      float* dst = S.raw + ((blk % 3) * kLB + (warp - 1)) * 1024;
      const float* src = th + (size_t)tstep(q) * mm;
      if (v16) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int e = lane + 32 * i;
          if (e < (mm >> 2)) cpa16(dst + 4 * e, src + 4 * e);
        }
      } else {
        for (int e = lane; e < mm; e += 32) cpa4(dst + e, src + e);
      }
    }
    cpa_commit();
  };
  auto convert = [&](int blk) {  // producers: raw block blk -> E = exp(theta) slots (warp w-1: step w-1)
    // No per-step max shift and no finiteness masks: anything the linear path cannot represent
    // (|theta| beyond the fp32 exp range, -inf structure that zeroes a state, NaN/+inf input) shows
    // up as a zero/non-finite state in the recurrence and sends the instance to the exact
    // log-space fallback.
    const int k = warp - 1;
    const int q = blk * kLB + k;
    if (q >= T) return;
    const float* r = S.raw + ((blk % 3) * kLB + k) * 1024;
    const int slot = q % kERing;
    float* E = S.E + slot * 32 * kEP;
    if (m == 32) {
#pragma unroll
      for (int a0 = 0; a0 < 32; a0 += 4) {  // rows a0..a0+3, lane = column b
        const float x0 = r[(a0 + 0) * 32 + lane], x1 = r[(a0 + 1) * 32 + lane];
        const float x2 = r[(a0 + 2) * 32 + lane], x3 = r[(a0 + 3) * 32 + lane];
        const float4 e = make_float4(ex2(x0 * SDB_LOG2E), ex2(x1 * SDB_LOG2E), ex2(x2 * SDB_LOG2E),
                                     ex2(x3 * SDB_LOG2E));
        if (dir == 0) {
          *reinterpret_cast<float4*>(E + lane * kEP + a0) = e;  // E^T[b][a0..a0+3]
        } else {
          E[(a0 + 0) * kEP + lane] = e.x;  // E[a][b]
          E[(a0 + 1) * kEP + lane] = e.y;
          E[(a0 + 2) * kEP + lane] = e.z;
          E[(a0 + 3) * kEP + lane] = e.w;
        }
      }
    } else {
      for (int a = 0; a < 32; ++a) {
        const float ev = (lane < m && a < m) ? ex2(r[a * m + lane] * SDB_LOG2E) : 0.f;
        if (dir == 0) E[lane * kEP + a] = ev;
        else E[a * kEP + lane] = ev;
      }
    }
    if (lane == 0) S.Mt[slot] = 0.f;
  };
  // ---- prologue
  if (warp > 0) {
    issue_raw(0);
    issue_raw(1);
    issue_raw(2);
    asm volatile("cp.async.wait_group 2;\n" ::);
    __syncwarp();
    convert(0);
  }
  // recurrence state (warp 0): linear vector v (lane holds component lane), scale
  float v = 0.f;
  double sc = 0.0;
  if (warp == 0) {
    if (dir == 0) {
      const float x = lane < m ? init[(size_t)b * m + lane] : ninf();
      if (lane < m && bad_input(x)) atomicOr(&flagsh, 1);
      const float mx = warp_max(x);
      const float mc = (mx == ninf()) ? 0.f : mx;
      v = lane < m ? fexp(x - mc) : 0.f;
      sc = (double)mc;
      if (lane < m) vecs[lane] = v;
      if (lane == 0) scs[0] = sc;
    } else {
      v = lane < m ? 1.f : 0.f;
      sc = 0.0;
      if (lane < m) vecs[(size_t)T * m + lane] = v;
      if (lane == 0) scs[T] = sc;
    }
    vsh[lane] = v;
  }
  __syncthreads();
  for (int blk = 0; blk < NB; ++blk) {
    if (warp == 0) {
      // ---------------- recurrence over the block
      for (int k = 0; k < kLB; ++k) {
        const int q = blk * kLB + k;
        if (q >= T) break;
        const int slot = q % kERing;
        const float* E = S.E + slot * 32 * kEP;
        // u_x = sum_y M[x][y] v_y: v broadcast from shared memory, both operands as float4
        const float4* vv = reinterpret_cast<const float4*>(vsh);
        const float4* row = reinterpret_cast<const float4*>(E + lane * kEP);
        float u0 = 0.f, u1 = 0.f, u2 = 0.f, u3 = 0.f;
#pragma unroll
        for (int y = 0; y < 8; ++y) {
          const float4 e4 = row[y], v4 = vv[y];
          u0 = fmaf(e4.x, v4.x, u0);
          u1 = fmaf(e4.y, v4.y, u1);
          u2 = fmaf(e4.z, v4.z, u2);
          u3 = fmaf(e4.w, v4.w, u3);
        }
        float u = (u0 + u1) + (u2 + u3);
        if (lane >= m) u = 0.f;
        // a zero or non-finite state (underflow/overflow of the linear form, -inf structure,
        // NaN/+inf input) -> exact log-space fallback for this instance
        if (lane < m && !(u > 0.f && u < __int_as_float(0x7f800000))) atomicOr(&flagsh, 2);
        // u >= 0: its float bits order like unsigned ints -> one REDUX for the max
        const float umax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(u)));
        float inv;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(umax));
        inv = umax > 0.f ? inv : 0.f;
        v = u * inv;
        __syncwarp();
        vsh[lane] = v;
        __syncwarp();
        // scale bookkeeping uses the factor actually applied (1/inv), so it is exact
        sc += (double)S.Mt[slot] + (umax > 0.f ? -(double)flog(inv) : 0.0);
        // the vector after processing position q belongs to step index (fwd) t+1 / (bwd) t
        const int tv = dir == 0 ? q + 1 : T - 1 - q;
        if (lane < m) vecs[(size_t)tv * m + lane] = v;
        if (lane == 0) scs[tv] = sc;
      }
    } else {
      // ---------------- producers: stage block blk+3, convert block blk+1, emit block blk-1
      issue_raw(blk + 3);
      asm volatile("cp.async.wait_group 2;\n" ::);
      __syncwarp();
      if (blk + 1 < NB) convert(blk + 1);
    }
    __syncthreads();
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  // ---------------- outputs.  Forward: log Z = c_T + log sum_a e_T[a] (beta_T = 0), status and
  // its verdict; backward: its verdict.  Anything but a clean linear result (invalid input, a
  // reachable state whose linear value underflowed or overflowed, vacuous) is recomputed by the
  // exact log-space path; the emission kernel merges the two verdicts.
  const int fl = flagsh;
  if (warp == 0) {
    const float tot = warp_sum(lane < m ? v : 0.f);
    if (lane == 0) {
      if (dir == 0) {
        const double Zf = (tot > 0.f && tot < __int_as_float(0x7f800000)) ? sc + (double)flog(tot) : ninfd();
        ws.need[b] = ((fl & 3) || Zf == ninfd()) ? 1 : 0;
        ws.flags[b] = SDB_ST_OK;
        status[b] = SDB_ST_OK;
        logz[b] = Zf;
      } else {
        ws.needb[b] = (fl & 3) ? 1 : 0;
      }
    }
  }
}

// marginals: grid (ceil((n-1)/kStepsPerBlock) + 1, B).  blockIdx.x == 0 also
// writes p_init.
constexpr int kStepsPerBlock = 8;

__global__ void __launch_bounds__(kThreads) chain_marg_kernel(
    const float* __restrict__ init, const float* __restrict__ trans, int n, int m, ChainWs ws,
    const double* __restrict__ logz, float* __restrict__ marg_init, float* __restrict__ marg_trans, int only_need) {
  const int b = blockIdx.y;
  if (only_need && ws.need[b] == 0) return;
  const int t0 = blockIdx.x * kStepsPerBlock;
  const size_t mm = (size_t)m * m;
  const bool ok = ws.flags[b] == SDB_ST_OK;
  const double z = logz[b];
  // exponent arguments summed in fp64: this kernel serves the log-space path, i.e. the instances
  // whose potentials are too large for the linear one (|theta| ~ 10^2: fp32 sums would cost 1e-4)
  if (blockIdx.x == 0 && marg_init) {
    const float* be = ws.beta + (size_t)b * n * m;
    const double K = ok ? ws.bcum[(size_t)b * n] - z : 0.0;
    for (int j = threadIdx.x; j < m; j += kThreads)
      marg_init[(size_t)b * m + j] = ok ? fexp((float)((double)init[(size_t)b * m + j] + (double)be[j] + K)) : 0.f;
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
    const double K = ws.acum[(size_t)b * n + t] + ws.bcum[(size_t)b * n + t + 1] - z;
    for (int e = threadIdx.x; e < (int)mm; e += kThreads) {
      const int a = e / m, j = e - a * m;
      out[e] = fexp((float)(((double)al[a] + K) + ((double)tt[e] + (double)be[j])));
    }
  }
}

// Marginals from the LINEAR passes (chain_lin_kernel): e_t, f_t normalised
// vectors with log scales c_t, d_t, so
//   p[t][a][b] = e_t[a] exp(theta_t[a][b]) f_(t+1)[b] exp(c_t + d_(t+1) - Z)
// (chain.py:84-95).  Grid (ceil((n-1)/kLinMargSteps), B), every element an
// independent streaming FMUL/MUFU -- HBM-bound.  Block (0, b) also writes
// p_init and merges the two passes' verdicts into ws.need[b]; instances that
// need the log-space path are skipped (chain_marg_kernel writes them).
constexpr int kLinMargSteps = 2;  // steps per CTA: short dependent load chains per thread

__global__ void __launch_bounds__(kThreads) chain_lin_marg_kernel(
    const float* __restrict__ init, const float* __restrict__ trans, int n, int m, ChainWs ws,
    const double* __restrict__ logz, float* __restrict__ marg_init, float* __restrict__ marg_trans) {
  const int b = blockIdx.y;
  const int need = ws.need[b] | ws.needb[b];
  if (blockIdx.x == 0 && threadIdx.x == 0) ws.need[b] = need;
  if (need) return;
  const double z = logz[b];
  const size_t mm = (size_t)m * m;
  const float* ev = ws.alpha + (size_t)b * n * m;
  const float* fv = ws.beta + (size_t)b * n * m;
  if (blockIdx.x == 0 && marg_init) {
    // p_init[a] = exp(init[a] + d_0 - Z) f_0[a]
    const float K = (float)(ws.bcum[(size_t)b * n] - z);
    for (int j = threadIdx.x; j < m; j += kThreads)
      marg_init[(size_t)b * m + j] = fexp(init[(size_t)b * m + j] + K) * fv[j];
  }
  if (!marg_trans) return;
  const int t0 = blockIdx.x * kLinMargSteps, t1 = min(t0 + kLinMargSteps, n - 1);
  for (int t = t0; t < t1; ++t) {
    const float* tt = trans + ((size_t)b * (n - 1) + t) * mm;
    float* out = marg_trans + ((size_t)b * (n - 1) + t) * mm;
    const float* e = ev + (size_t)t * m;
    const float* f = fv + (size_t)(t + 1) * m;
    const float K = (float)(ws.acum[(size_t)b * n + t] + ws.bcum[(size_t)b * n + t + 1] - z);
    if ((m & 3) == 0) {
      const float4* t4 = reinterpret_cast<const float4*>(tt);
      float4* o4 = reinterpret_cast<float4*>(out);
      const int m4 = m >> 2;
      const int sh = ((m4 & (m4 - 1)) == 0) ? __ffs(m4) - 1 : -1;  // m4 a power of two: shift, no division
      for (int x = threadIdx.x; x < (int)(mm >> 2); x += kThreads) {
        const int a = sh >= 0 ? (x >> sh) : x / m4, j = (x - a * m4) * 4;
        const float ea = e[a];
        const float4 v = __ldg(t4 + x);
        float4 r;
        r.x = fexp(v.x + K) * ea * f[j + 0];
        r.y = fexp(v.y + K) * ea * f[j + 1];
        r.z = fexp(v.z + K) * ea * f[j + 2];
        r.w = fexp(v.w + K) * ea * f[j + 3];
        o4[x] = r;
      }
    } else {
      for (int x = threadIdx.x; x < (int)mm; x += kThreads) {
        const int a = x / m, j = x - a * m;
        out[x] = fexp(tt[x] + K) * e[a] * f[j];
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

// Viterbi fast path (m <= 32), one CTA of 256 threads per instance and ONE
// barrier per step.  Thread (warp w, lane l) owns next tag b = 4w + (l & 3)
// and the predecessors a = ag + 8q (ag = l >> 2, q = 0..3, ascending, strict
// '>' = first maximum); the 8 predecessor groups of a tag are lanes l ^ 4,
// l ^ 8, l ^ 16, merged by three shuffles with the (value, lower index) rule
// -- identical tie semantics to chain.py:106 and the reference's addition
// order (score[a] + theta[a, b] in float64).  Potentials stream through a
// (kD+1)-slot cp.async ring (rows at a 36-float pitch: the 32 lanes of a
// warp read 32 distinct banks); the scores are double-buffered, so the barrier
// at the top of a step both publishes the previous scores and frees the ring
// slot refilled in this step.
constexpr int kVP = 36;  // ring row pitch (floats)

__global__ void __launch_bounds__(kThreads) chain_viterbi_small_kernel(
    const float* __restrict__ init, const float* __restrict__ trans, int n, int m, int32_t* __restrict__ tags,
    double* __restrict__ score, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) float smv[];
  const int mm = m * m, slot = m * kVP;
  float* ring = smv;                                                  // [kD+1][m][kVP]
  double* dl = reinterpret_cast<double*>(ring + (kD + 1) * slot);     // [2][32]
  uint8_t* back = reinterpret_cast<uint8_t*>(dl + 64);                // [n][32]
  __shared__ int redi[kThreads / 32];
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tb = 4 * warp + (lane & 3), ag = lane >> 2;
  const float* th = trans + (size_t)b * (n - 1) * mm;
  const bool v16 = ((m & 3) == 0) && ((((uintptr_t)th) & 15) == 0);
  // this thread's 16-byte chunk of a step (m <= 32: m*m/4 <= 256 chunks), fixed for all steps
  const int q4 = m >> 2;
  const int cr = q4 ? tid / q4 : 0, cc = tid - cr * q4;
  const bool has16 = v16 && tid < m * q4;
  const int soff = cr * m + 4 * cc, doff = cr * kVP + 4 * cc;
  auto stage = [&](int t, int sl) {
    float* d = ring + sl * slot;
    const float* src = th + (size_t)t * mm;
    if (v16) {
      if (has16) cpa16(d + doff, src + soff);
    } else {
      for (int e = tid; e < mm; e += kThreads) {
        const int r = e / m, c = e - r * m;
        cpa4(d + r * kVP + c, src + e);
      }
    }
  };
  for (int d = 0; d < kD; ++d) {
    if (d < n - 1) stage(d, d);
    cpa_commit();
  }
  int bad = 0;
  if (tid < 32) {
    const float x = tid < m ? init[(size_t)b * m + tid] : ninf();
    bad |= (tid < m) && bad_input(x);
    dl[tid] = tid < m ? (double)x : ninfd();
  }
  const bool bok = tb < m;
  int rsl = 0, wsl = kD;  // ring slots read / refilled this step
  for (int t = 0; t < n - 1; ++t) {
    cpa_wait_d();
    __syncthreads();
    const double* cur = dl + (t & 1) * 32;
    double* nxt = dl + ((t + 1) & 1) * 32;
    const float* tt = ring + rsl * slot;
    float x[4];
    double d[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int a = ag + 8 * q;
      const int ac = a < m ? a : 0;
      x[q] = tt[ac * kVP + (bok ? tb : 0)];
      d[q] = cur[ac];
    }
    if (t + kD < n - 1) stage(t + kD, wsl);
    cpa_commit();
    rsl = rsl == kD ? 0 : rsl + 1;
    wsl = wsl == kD ? 0 : wsl + 1;
    double best = ninfd();
    int arg = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int a = ag + 8 * q;
      const bool live = bok && a < m;
      bad |= live && bad_input(x[q]);
      const double v = live ? d[q] + (double)x[q] : ninfd();
      if (v > best) { best = v; arg = live ? a : arg; }
    }
#pragma unroll
    for (int o = 4; o <= 16; o <<= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
      if (ov > best || (ov == best && oa < arg)) { best = ov; arg = oa; }
    }
    if (ag == 0 && bok) {
      nxt[tb] = best;
      back[(size_t)(t + 1) * 32 + tb] = (uint8_t)(arg == 0x7fffffff ? 0 : arg);
    } else if (ag == 0 && tb < 32) {
      nxt[tb] = ninfd();
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  bad = block_or(bad, redi);  // (contains the barrier that publishes the last scores)
  if (warp == 0) {
    const double* fin = dl + ((n - 1) & 1) * 32;
    double best = lane < m ? fin[lane] : ninfd();
    int arg = lane < m ? lane : 0x7fffffff;
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
      if (ov > best || (ov == best && oa < arg)) { best = ov; arg = oa; }
    }
    __syncwarp();
    if (lane == 0) {
      int32_t* tg = tags + (size_t)b * n;
      const bool vac = (best == ninfd());
      status[b] = bad ? SDB_ST_INVALID : (vac ? SDB_ST_VACUOUS : SDB_ST_OK);
      score[b] = best;
      int cur = vac ? 0 : arg;
      tg[n - 1] = cur;
      for (int t = n - 2; t >= 0; --t) {
        cur = vac ? 0 : back[(size_t)(t + 1) * 32 + cur];
        tg[t] = cur;
      }
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
  const bool lin = (m <= 32) && (n - 1 >= 2 * kLB);
  const size_t small_smem = (size_t)kD * m * m * 4 + (32 + 2 * kGroups * 32) * 4;
  if (lin) {
    const size_t smem = lin_smem_bytes();
    if (cudaFuncSetAttribute(chain_lin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SDB_ERR_CUDA;
    chain_lin_kernel<<<(unsigned)(2 * B), kThreads, smem, s>>>(init, trans, n, m, ws, logz, status);
    SDB_CHECK_LAUNCH();
    // marginals of the linear instances (also merges the two passes' verdicts into ws.need)
    dim3 gl((unsigned)((n - 1 + kLinMargSteps - 1) / kLinMargSteps), (unsigned)B);
    chain_lin_marg_kernel<<<gl, kThreads, 0, s>>>(init, trans, n, m, ws, logz, marg_init, marg_trans);
    dim3 g((unsigned)((n - 1 + kStepsPerBlock - 1) / kStepsPerBlock), (unsigned)B);
    SDB_CHECK_LAUNCH();
    // exact log-space recomputation of the (rare) instances the linear path flagged
    if (cudaFuncSetAttribute(chain_fwd_bwd_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)small_smem) != cudaSuccess)
      return SDB_ERR_CUDA;
    chain_fwd_bwd_small_kernel<<<dim3((unsigned)B, 2), kThreads, small_smem, s>>>(init, trans, n, m, ws, logz,
                                                                                  status, 1);
    SDB_CHECK_LAUNCH();
    if (marg_init || marg_trans) {
      chain_marg_kernel<<<g, kThreads, 0, s>>>(init, trans, n, m, ws, logz, marg_init, marg_trans, 1);
      SDB_CHECK_LAUNCH();
    }
    return SDB_OK;
  }
  if (m <= 32) {
    if (cudaFuncSetAttribute(chain_fwd_bwd_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)small_smem) != cudaSuccess)
      return SDB_ERR_CUDA;
    chain_fwd_bwd_small_kernel<<<dim3((unsigned)B, 2), kThreads, small_smem, s>>>(init, trans, n, m, ws, logz,
                                                                                  status, 0);
  } else {
    size_t smem = (size_t)m * 4 * (1 + 2 * kGroups);
    if (smem > 48 * 1024) {
      if (cudaFuncSetAttribute(chain_fwd_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
        return SDB_ERR_CUDA;
    }
    chain_fwd_bwd_kernel<<<dim3((unsigned)B, 2), kThreads, smem, s>>>(init, trans, n, m, ws, logz, status);
  }
  SDB_CHECK_LAUNCH();
  if (marg_init || marg_trans) {
    dim3 g((unsigned)((n - 1 + kStepsPerBlock - 1) / kStepsPerBlock + (n == 1 ? 1 : 0)), (unsigned)B);
    chain_marg_kernel<<<g, kThreads, 0, s>>>(init, trans, n, m, ws, logz, marg_init, marg_trans, 0);
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
  if (m <= 32) {
    const size_t smem = (size_t)(kD + 1) * m * kVP * 4 + 64 * 8 + (size_t)n * 32 + 64;
    if (smem <= 200 * 1024) {
      if (cudaFuncSetAttribute(chain_viterbi_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
        return SDB_ERR_CUDA;
      chain_viterbi_small_kernel<<<(unsigned)B, kThreads, smem, (cudaStream_t)stream>>>(init, trans, n, m, tags,
                                                                                       score, status);
      SDB_CHECK_LAUNCH();
      return SDB_OK;
    }
  }
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
