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

#include <cooperative_groups.h>

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

// one log-space pass (forward or backward) of instance b by the whole CTA; the marginals are
// formed from the stored normalised vectors by marg_steps().  `sm` >= kD*m*m + (32 + 2*kGroups*32) floats.
__device__ void small_pass(const float* __restrict__ init, const float* __restrict__ trans, int n, int m,
                           const ChainWs& ws, double* __restrict__ logz, int32_t* __restrict__ status, int b,
                           bool fwd, float* sm, int nl = -1) {
  // n: this instance's length; nl: the layout length of the batch (strides), >= n
  if (nl < 0) nl = n;
  const int mm = m * m;
  float* stage = sm;                     // [kD][mm]
  float* vec = stage + kD * mm;          // [32]
  float* pm = vec + 32;                  // [kGroups][32]
  float* ps = pm + kGroups * 32;         // [kGroups][32]
  __shared__ int redi[kThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* th = trans + (size_t)b * (nl - 1) * mm;
  const bool v16 = ((mm & 3) == 0);
  int bad = 0;
  // prologue prefetch: steps in processing order
  for (int d = 0; d < kD; ++d) {
    const int t = fwd ? d : n - 2 - d;
    if (d < n - 1) stage_step(stage + d * mm, th + (size_t)t * mm, mm, v16);
    cpa_commit();
  }
  if (fwd) {
    float* al = ws.alpha + (size_t)b * nl * m;
    double* ac = ws.acum + (size_t)b * nl;
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
    float* be = ws.beta + (size_t)b * nl * m;
    double* bc = ws.bcum + (size_t)b * nl;
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

__global__ void __launch_bounds__(kThreads) chain_fwd_bwd_small_kernel(
    const float* __restrict__ init, const float* __restrict__ trans, int n, int m, ChainWs ws,
    double* __restrict__ logz, int32_t* __restrict__ status, int only_need) {
  if (only_need && ws.need[blockIdx.x] == 0) return;
  extern __shared__ __align__(16) float sm_small[];
  small_pass(init, trans, n, m, ws, logz, status, blockIdx.x, blockIdx.y == 0, sm_small);
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

// marginals of steps [t0, t1) of instance b from the log-space passes' vectors (+ p_init if asked)
__device__ void marg_steps(const float* __restrict__ init, const float* __restrict__ trans, int n, int m,
                           const ChainWs& ws, const double* __restrict__ logz, float* __restrict__ marg_init,
                           float* __restrict__ marg_trans, int b, int t0, int t1, bool with_init) {
  const size_t mm = (size_t)m * m;
  const bool ok = ws.flags[b] == SDB_ST_OK;
  const double z = logz[b];
  // exponent arguments summed in fp64: this kernel serves the log-space path, i.e. the instances
  // whose potentials are too large for the linear one (|theta| ~ 10^2: fp32 sums would cost 1e-4)
  if (with_init && marg_init) {
    const float* be = ws.beta + (size_t)b * n * m;
    const double K = ok ? ws.bcum[(size_t)b * n] - z : 0.0;
    for (int j = threadIdx.x; j < m; j += kThreads)
      marg_init[(size_t)b * m + j] = ok ? fexp((float)((double)init[(size_t)b * m + j] + (double)be[j] + K)) : 0.f;
  }
  if (!marg_trans) return;
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

__global__ void __launch_bounds__(kThreads) chain_marg_kernel(
    const float* __restrict__ init, const float* __restrict__ trans, int n, int m, ChainWs ws,
    const double* __restrict__ logz, float* __restrict__ marg_init, float* __restrict__ marg_trans, int only_need) {
  const int b = blockIdx.y;
  if (only_need && ws.need[b] == 0) return;
  const int t0 = blockIdx.x * kStepsPerBlock;
  marg_steps(init, trans, n, m, ws, logz, marg_init, marg_trans, b, t0, min(t0 + kStepsPerBlock, n - 1),
             blockIdx.x == 0);
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

// ---------------------------------------------------------------------
// Time-parallel chain scan (m <= 32): log_partition + marginals in ONE
// cluster launch (chain.py:64-95).
//
// The T = n-1 transition steps are cut into kSC chunks; the kSC CTAs of a
// thread-block cluster own one chunk each of one instance.  Linear space with
// exact power-of-two normalisers (log scales are integers x ln2 plus the
// per-step shifts, summed in fp64):
//   A  stage the chunk's potentials with bulk TMA copies (cp.async.bulk, one
//      per step, mbarrier completion), E_t = exp(theta_t - max theta_t)
//      (swizzled 16-byte granules: row and column reads are conflict-free),
//      and the chunk's transfer product P_c = E_t0 E_t0+1 ... (a 32x32x32
//      FFMA product per step; each thread owns 4 rows x 1 column);
//   B  after a cluster barrier every CTA copies the other chunks' P~ through
//      distributed shared memory and folds them into its boundary vectors:
//      alpha at its chunk start (warp 0) and beta at its chunk end (warp 1);
//   C  recompute alpha / beta inside the chunk (warp 0 forward, warp 1
//      backward -- the reverse scan, no autodiff), then emit
//      p_t[a][b] = alpha~_t[a] E_t[a][b] beta~_t+1[b] e^K_t as float4 rows.
// Numerical guard: a chunk whose potentials span more than 80 nats within a
// step (exp would underflow), a zero normaliser, an out-of-range marginal
// scale or a NaN/+inf input sends the WHOLE instance to the exact log-space
// path, run inline by the cluster's rank-0 CTA (small_pass + marg_steps).
#ifdef SDB_SCAN_PROF
__device__ unsigned long long g_scan_t[1024][10];
#define SCAN_TS(i)                                                                     \
  do {                                                                                 \
    if (threadIdx.x == 0 && blockIdx.x < 1024) {                                       \
      g_scan_t[blockIdx.x][i] = clock64();                                             \
    }                                                                                  \
  } while (0)
#else
#define SCAN_TS(i) \
  do {             \
  } while (0)
#endif
constexpr int kSC = 8;                    // chunks per instance = cluster size
constexpr int kW = kThreads / 32;
constexpr int kSLmax = 24;                // steps per chunk (shared-memory bound)
constexpr int kXP = 36;                   // pitch of the transposed product (conflict-free float4 stores)
constexpr float kRange = 80.f;            // max nats inside one step before linear space gives up

__device__ __forceinline__ int swz(int a, int b) { return (a << 5) + ((((b >> 2) ^ (a & 7))) << 2) + (b & 3); }
// column b's offset inside a swizzled row whose index is congruent to q mod 8
__device__ __forceinline__ int swc(int q, int b) { return (((b >> 2) ^ q) << 2) + (b & 3); }
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(const uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
}

struct ScanSmem {
  float* E;        // [L][1024] raw theta, then E (swizzled)
  float* XT;       // [2][32][kXP] product, transposed (XT[k][r] = Y[r][k])
  float* P;        // [1024] own normalised chunk product (swizzled; read by the other ranks)
  float* al;       // [L+1][32] alpha~ within the chunk
  float* be;       // [L+1][32] beta~ within the chunk
  float* vec;      // [2][32] boundary-scan vectors (alpha, beta)
  float* gh;       // [L] emission factor e^(K_t / 2)
  double* la;      // [L+1] log scales of al
  double* lb;      // [L+1] log scales of be
  double* lpc;     // [kSC] log scale of each chunk's product
  float* mx;       // [L] step max
  int* pe;         // [2][kW] power-of-two exponents of the warp maxima (double-buffered)
  uint64_t* mbar;  // [L] TMA completion
  uint64_t* rdy;   // [L] converted tile ready (32 arrivals)
  int* flagA;      // [kSC] phase-A verdicts pushed by every rank
  int* flagC;      // [kSC] phase-C verdicts
  double* misc;    // [4] logZ, ...
};

size_t scan_smem(int L) {
  return (size_t)L * 4096 + 2 * 32 * kXP * 4 + 4096 + 2 * (L + 1) * 32 * 4 + 2 * 32 * 4 + L * 4 +
         2 * (L + 1) * 8 + kSC * 8 + L * 4 + 2 * 8 * 4 + 2 * L * 8 + 2 * kSC * 4 + 4 * 8 + 32 * 16;
}

__device__ __forceinline__ ScanSmem scan_carve(char* p, int L) {
  ScanSmem S;
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 15) & ~(size_t)15;
    return r;
  };
  S.E = (float*)take((size_t)L * 4096);
  S.XT = (float*)take(2 * 32 * kXP * 4);
  S.P = (float*)take(4096);
  S.al = (float*)take((size_t)(L + 1) * 32 * 4);
  S.be = (float*)take((size_t)(L + 1) * 32 * 4);
  S.vec = (float*)take(2 * 32 * 4);
  S.gh = (float*)take((size_t)L * 4);
  S.la = (double*)take((size_t)(L + 1) * 8);
  S.lb = (double*)take((size_t)(L + 1) * 8);
  S.lpc = (double*)take(kSC * 8);
  S.mx = (float*)take((size_t)L * 4);
  S.pe = (int*)take(2 * 8 * 4);
  S.mbar = (uint64_t*)take((size_t)L * 8);
  S.rdy = (uint64_t*)take((size_t)L * 8);
  S.flagA = (int*)take(kSC * 4);
  S.flagC = (int*)take(kSC * 4);
  S.misc = (double*)take(4 * 8);
  return S;
}

// exponent e with 2^e <= x < 2^(e+1) for a positive normal float (0 for x == 0 / denormal)
__device__ __forceinline__ int fexpo(float x) { return (int)((__float_as_uint(x) >> 23) & 0xff) - 127; }

template <bool kFull>  // kFull: m == 32 (bulk TMA staging); else padded element loads
__global__ void __launch_bounds__(kThreads, 2) chain_scan_kernel(
    const float* __restrict__ init, const float* __restrict__ trans, int n, int m, ChainWs ws,
    double* __restrict__ logz, float* __restrict__ marg_init, float* __restrict__ marg_trans,
    int32_t* __restrict__ status, const int32_t* __restrict__ lengths) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) char smscan[];
  // per-instance length (ragged batches, chain.py:161-176 without padding): this instance
  // has T = lengths[b] - 1 steps; the arrays keep the batch layout of Tl = n - 1 steps
  const int b = blockIdx.x / kSC;
  const int Tl = n - 1, T = lengths ? min(max(lengths[b], 1), n) - 1 : Tl, L = (T + kSC - 1) / kSC;
  ScanSmem S = scan_carve(smscan, L);
  const int c = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t0 = min(T, c * L), t1 = min(T, t0 + L), Lc = t1 - t0;
  const float* th = trans + ((size_t)b * Tl + t0) * (size_t)(m * m);
  const float LN2 = 0.6931471805599453f;

  SCAN_TS(0);
  // ---- A0: stage the chunk (bulk TMA per step, or padded loads) ----------------------------
  if (tid == 0) {
    for (int k = 0; k < Lc; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(smem_u32(S.rdy + k)));
    if (!kFull) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (kFull) {
    if (tid == 0) {
      for (int k = 0; k < Lc; ++k)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(S.mbar + k)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int k = 0; k < Lc; ++k) {
        const uint32_t bar = smem_u32(S.mbar + k);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" ::"r"(bar) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];"
                     ::"r"(smem_u32(S.E + k * 1024)), "l"(th + (size_t)k * 1024), "r"(bar) : "memory");
      }
    }
  } else {
    for (int e = tid; e < Lc * 1024; e += kThreads) {
      const int k = e >> 10, a = (e >> 5) & 31, bb = e & 31;
      S.E[e] = (a < m && bb < m) ? __ldg(th + (size_t)k * m * m + a * m + bb) : ninf();
    }
  }
  if (tid < kSC) { S.flagA[tid] = 0; S.flagC[tid] = 0; }
  __syncthreads();

  // ---- A: warps 4-7 convert tiles (E_t = exp(theta_t - mx_t), one row per lane, swizzled in
  // place) in step order and release each through an mbarrier; warps 0-3 multiply as tiles
  // become ready (Y_k = Y~_(k-1) E_k, a 4 x 2 output block per lane, normalised by powers of two)
  int flag = 0;
  int esum = 0;  // product warps: sum of normaliser exponents
  int cur = 0;
  if (warp >= 4) {
    if (warp == kW - 1) {  // alpha_0 = exp(init - max init) (every rank needs it for its boundary vector)
      const float x = lane < m ? init[(size_t)b * m + lane] : ninf();
      const float mi = warp_max(x);
      float lo = x == ninf() ? __int_as_float(0x7f800000) : x;
      lo = -warp_max(-lo);
      if (__any_sync(0xffffffffu, bad_input(x)) || mi == ninf() || mi - lo > kRange) flag = 1;
      S.vec[lane] = lane < m ? fexp(x - (mi == ninf() ? 0.f : mi)) : 0.f;
      if (lane == 0) S.misc[1] = (double)mi;  // log scale of alpha~_0
    }
    for (int k = warp - 4; k < Lc; k += 4) {
      if (kFull) mbar_wait(S.mbar + k, 0);
      float* tile = S.E + k * 1024;
      float4 v[8];
#pragma unroll
      for (int g = 0; g < 8; ++g) v[g] = *reinterpret_cast<const float4*>(tile + lane * 32 + 4 * ((g + lane) & 7));
      float hi = ninf(), lo = __int_as_float(0x7f800000);
      int bad = 0;
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const float q[4] = {v[g].x, v[g].y, v[g].z, v[g].w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          bad |= bad_input(q[u]);
          hi = fmaxf(hi, q[u]);
          if (q[u] != ninf()) lo = fminf(lo, q[u]);
        }
      }
      const float mxk = warp_max(hi);
      const float mnk = -warp_max(-lo);
      if (__any_sync(0xffffffffu, bad) || mxk == ninf() || mxk - mnk > kRange) flag = 1;
      const float sh = mxk == ninf() ? 0.f : mxk;
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const int gl = (g + lane) & 7;  // logical granule held in v[g]
        float4 e;
        e.x = fexp(v[g].x - sh);
        e.y = fexp(v[g].y - sh);
        e.z = fexp(v[g].z - sh);
        e.w = fexp(v[g].w - sh);
        *reinterpret_cast<float4*>(tile + lane * 32 + 4 * (gl ^ (lane & 7))) = e;
      }
      if (lane == 0) S.mx[k] = mxk;
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(S.rdy + k)) : "memory");
    }
  } else {
    const int pt = tid;  // 0..127
    // Y_0 = E_t0 (max 1): transposed copy
    if (Lc > 0) mbar_wait(S.rdy, 0);
    for (int e = pt; e < 1024; e += 128) {
      const int r = e >> 5, j = e & 31;
      S.XT[j * kXP + r] = Lc > 0 ? S.E[swz(r, j)] : (r == j ? 1.f : 0.f);
    }
    if (pt < 4) S.pe[pt] = 0;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    SCAN_TS(1);
    const int rb = (warp >> 1) * 16 + 4 * (lane >> 3);  // first of this lane's 4 rows
    const int cb = (warp & 1) * 16 + 2 * (lane & 7);    // first of its 2 columns
    int co[8];                                          // column offset inside a swizzled row, per row & 7
#pragma unroll
    for (int q = 0; q < 8; ++q) co[q] = swc(q, cb);
    for (int k = 1; k < Lc; ++k) {
      const float* X = S.XT + cur * 32 * kXP;
      const float* Ek = S.E + k * 1024;
      int emax = max(max(S.pe[cur * 4], S.pe[cur * 4 + 1]), max(S.pe[cur * 4 + 2], S.pe[cur * 4 + 3]));
      mbar_wait(S.rdy + k, 0);
      float acc[4][2] = {};
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float4 x = *reinterpret_cast<const float4*>(X + j * kXP + rb);
        const float2 e = *reinterpret_cast<const float2*>(Ek + j * 32 + co[j & 7]);
        acc[0][0] = fmaf(x.x, e.x, acc[0][0]);
        acc[0][1] = fmaf(x.x, e.y, acc[0][1]);
        acc[1][0] = fmaf(x.y, e.x, acc[1][0]);
        acc[1][1] = fmaf(x.y, e.y, acc[1][1]);
        acc[2][0] = fmaf(x.z, e.x, acc[2][0]);
        acc[2][1] = fmaf(x.z, e.y, acc[2][1]);
        acc[3][0] = fmaf(x.w, e.x, acc[3][0]);
        acc[3][1] = fmaf(x.w, e.y, acc[3][1]);
      }
      const float sc = __int_as_float((127 - emax) << 23);  // 2^-emax (exact)
      esum += emax;
      float mxl = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[i][0] *= sc;
        acc[i][1] *= sc;
        mxl = fmaxf(mxl, fmaxf(acc[i][0], acc[i][1]));
      }
      const float wm = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(mxl)));
      const int nx = cur ^ 1;
      float* Xn = S.XT + nx * 32 * kXP;
      *reinterpret_cast<float4*>(Xn + cb * kXP + rb) = make_float4(acc[0][0], acc[1][0], acc[2][0], acc[3][0]);
      *reinterpret_cast<float4*>(Xn + (cb + 1) * kXP + rb) = make_float4(acc[0][1], acc[1][1], acc[2][1], acc[3][1]);
      if (lane == 0) S.pe[nx * 4 + warp] = wm > 0.f ? fexpo(wm) : -1000;
      cur = nx;
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    int emax = max(max(S.pe[cur * 4], S.pe[cur * 4 + 1]), max(S.pe[cur * 4 + 2], S.pe[cur * 4 + 3]));
    if (emax < -120) flag = 1;  // the product underflowed
    emax = max(emax, -120);
    const float sc = __int_as_float((127 - emax) << 23);
    esum += emax;
    const float* X = S.XT + cur * 32 * kXP;
    for (int e = pt; e < 1024; e += 128) {
      const int r = e >> 5, j = e & 31;
      S.P[swz(r, j)] = X[j * kXP + r] * sc;
    }
  }
  __syncthreads();
  SCAN_TS(2);
  int sw[8];  // this lane's column inside a swizzled row, per row residue (row & 7)
#pragma unroll
  for (int q = 0; q < 8; ++q) sw[q] = swc(q, lane);
  if (tid == 0) {
    double lp = (double)esum * (double)LN2;
    for (int k = 0; k < Lc; ++k) lp += (double)S.mx[k];
    S.lpc[c] = lp;
  }
  const int anyA = __syncthreads_or(flag);
  if (tid < kSC) *cluster.map_shared_rank(S.flagA + c, tid) = anyA;  // push the verdict to every rank
  cluster.sync();  // #1: every chunk product, scale and verdict visible cluster-wide
  SCAN_TS(3);

  int fail = 0;
#pragma unroll
  for (int r = 0; r < kSC; ++r) fail |= S.flagA[r];
  if (fail) goto fallback;
  {
    // ---- B: fold the other chunks' products (read in place through DSMEM) into the boundary
    // vectors
    if (tid < kSC && tid != c) S.lpc[tid] = *cluster.map_shared_rank(S.lpc + tid, tid);
    __syncthreads();
    if (warp == 0) {
      // alpha at the chunk start: alpha~_0 P~_0 ... P~_(c-1)  (lane = column b)
      float* v = S.vec;
      double A = S.misc[1];
      for (int j = 0; j < c; ++j) {
        const float* Pj = cluster.map_shared_rank(S.P, j);
        float pr[32];
#pragma unroll
        for (int a = 0; a < 32; ++a) pr[a] = Pj[a * 32 + sw[a & 7]];
        float acc4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int a = 0; a < 32; a += 4) {
          const float4 vv = *reinterpret_cast<const float4*>(v + a);
          acc4[0] = fmaf(vv.x, pr[a], acc4[0]);
          acc4[1] = fmaf(vv.y, pr[a + 1], acc4[1]);
          acc4[2] = fmaf(vv.z, pr[a + 2], acc4[2]);
          acc4[3] = fmaf(vv.w, pr[a + 3], acc4[3]);
        }
        const float acc = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
        const float wm = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(acc)));
        const int ex = wm > 0.f ? fexpo(wm) : -1000;
        if (ex < -120) flag = 1;
        __syncwarp();
        v[lane] = acc * __int_as_float((127 - max(ex, -120)) << 23);
        __syncwarp();
        A += (double)max(ex, -120) * (double)LN2 + S.lpc[j];
      }
      S.al[lane] = v[lane];
      if (lane == 0) S.la[0] = A;
    } else if (warp == 1) {
      // beta at the chunk end: P~_(c+1) ... P~_(C-1) 1  (lane = row a)
      float* w = S.vec + 32;
      w[lane] = lane < m ? 1.f : 0.f;
      __syncwarp();
      double Bv = 0.0;
      for (int j = kSC - 1; j > c; --j) {
        const float* Pj = cluster.map_shared_rank(S.P, j);
        float4 pr[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) pr[g] = *reinterpret_cast<const float4*>(Pj + lane * 32 + 4 * (g ^ (lane & 7)));
        float acc4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          const float4 ww = *reinterpret_cast<const float4*>(w + 4 * g);
          acc4[0] = fmaf(pr[g].x, ww.x, acc4[0]);
          acc4[1] = fmaf(pr[g].y, ww.y, acc4[1]);
          acc4[2] = fmaf(pr[g].z, ww.z, acc4[2]);
          acc4[3] = fmaf(pr[g].w, ww.w, acc4[3]);
        }
        const float acc = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
        const float wm = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(acc)));
        const int ex = wm > 0.f ? fexpo(wm) : -1000;
        if (ex < -120) flag = 1;
        __syncwarp();
        w[lane] = acc * __int_as_float((127 - max(ex, -120)) << 23);
        __syncwarp();
        Bv += (double)max(ex, -120) * (double)LN2 + S.lpc[j];
      }
      S.be[Lc * 32 + lane] = w[lane];
      if (lane == 0) S.lb[Lc] = Bv;
    }
    __syncthreads();
    SCAN_TS(4);
    // ---- C: alpha / beta inside the chunk (warp 0 forward, warp 1 backward) ----------------
    if (warp == 0) {
      double A = S.la[0];
      for (int k = 0; k < Lc; ++k) {
        const float* Ek = S.E + k * 1024;
        const float* v = S.al + k * 32;
        float acc4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int a = 0; a < 32; a += 4) {
          const float4 vv = *reinterpret_cast<const float4*>(v + a);
          acc4[0] = fmaf(vv.x, Ek[a * 32 + sw[a & 7]], acc4[0]);
          acc4[1] = fmaf(vv.y, Ek[(a + 1) * 32 + sw[(a + 1) & 7]], acc4[1]);
          acc4[2] = fmaf(vv.z, Ek[(a + 2) * 32 + sw[(a + 2) & 7]], acc4[2]);
          acc4[3] = fmaf(vv.w, Ek[(a + 3) * 32 + sw[(a + 3) & 7]], acc4[3]);
        }
        const float acc = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
        const float wm = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(acc)));
        const int ex = wm > 0.f ? fexpo(wm) : -1000;
        if (ex < -120) flag = 1;
        S.al[(k + 1) * 32 + lane] = acc * __int_as_float((127 - max(ex, -120)) << 23);
        A += (double)max(ex, -120) * (double)LN2 + (double)S.mx[k];
        if (lane == 0) S.la[k + 1] = A;
        __syncwarp();
      }
#ifdef SDB_SCAN_PROF
      if (lane == 0) g_scan_t[blockIdx.x][8] = clock64();
#endif
    } else if (warp == 1) {
      double Bv = S.lb[Lc];
      for (int k = Lc - 1; k >= 0; --k) {
        const float* Ek = S.E + k * 1024;
        const float* w = S.be + (k + 1) * 32;
        float acc4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          const float4 er = *reinterpret_cast<const float4*>(Ek + lane * 32 + 4 * (g ^ (lane & 7)));
          const float4 ww = *reinterpret_cast<const float4*>(w + 4 * g);
          acc4[0] = fmaf(er.x, ww.x, acc4[0]);
          acc4[1] = fmaf(er.y, ww.y, acc4[1]);
          acc4[2] = fmaf(er.z, ww.z, acc4[2]);
          acc4[3] = fmaf(er.w, ww.w, acc4[3]);
        }
        const float acc = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
        const float wm = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(acc)));
        const int ex = wm > 0.f ? fexpo(wm) : -1000;
        if (ex < -120) flag = 1;
        S.be[k * 32 + lane] = acc * __int_as_float((127 - max(ex, -120)) << 23);
        Bv += (double)max(ex, -120) * (double)LN2 + (double)S.mx[k];
        if (lane == 0) S.lb[k] = Bv;
        __syncwarp();
      }
#ifdef SDB_SCAN_PROF
      if (lane == 0) g_scan_t[blockIdx.x][9] = clock64();
#endif
    }
    __syncthreads();
    SCAN_TS(5);
    // log Z from this chunk's start: A_t0 + B_t0 + log sum_a alpha~ beta~, and the emission factors
    if (warp == 0) {
      const float z = S.al[lane] * S.be[lane];
      const float zs = warp_sum(z);
      if (!(zs > 0.f)) flag = 1;
      const double lz = S.la[0] + S.lb[0] + (double)flog(fmaxf(zs, 1e-38f));
      if (lane == 0) S.misc[0] = lz;
      for (int k = lane; k < Lc; k += 32) {
        const double K = S.la[k] + (double)S.mx[k] + S.lb[k + 1] - lz;  // p = al E be e^K
        if (K > 170.0) flag = 1;
        S.gh[k] = fexp((float)(0.5 * fmin(K, 170.0)));
      }
    }
    const int anyC = __syncthreads_or(flag);
    if (tid < kSC) *cluster.map_shared_rank(S.flagC + c, tid) = anyC;
  }
  SCAN_TS(6);
  cluster.sync();  // #2: no rank reads another's shared memory after this
  SCAN_TS(7);
  {
    int failc = 0;
#pragma unroll
    for (int r = 0; r < kSC; ++r) failc |= S.flagC[r];
    if (failc) goto fallback;
  }
  // ---- emission: p_t[a][b] = (alpha~[a] g) E[a][b] (beta~[b] g) --------------------------
  if (c == 0 && tid == 0) {
    logz[b] = S.misc[0];
    status[b] = SDB_ST_OK;
  }
  if (marg_init && c == 0 && tid < m) {
    const double K = S.la[0] + S.lb[0] - S.misc[0];
    marg_init[(size_t)b * m + tid] = (float)((double)(S.al[tid] * S.be[tid]) * exp(K));
  }
  if (marg_trans) {
    // steps past this instance's length: marginal 0
    for (size_t e = (size_t)T * m * m + (size_t)c * kThreads + tid; e < (size_t)Tl * m * m;
         e += (size_t)kSC * kThreads)
      marg_trans[(size_t)b * Tl * m * m + e] = 0.f;
    float* out = marg_trans + ((size_t)b * Tl + t0) * (size_t)(m * m);
    if (kFull) {
      const int a = tid >> 3, g = tid & 7;
      for (int k = 0; k < Lc; ++k) {
        const float gk = S.gh[k];
        const float ra = S.al[k * 32 + a] * gk;
        const float4 e = *reinterpret_cast<const float4*>(S.E + k * 1024 + a * 32 + 4 * (g ^ (a & 7)));
        const float4 bv = *reinterpret_cast<const float4*>(S.be + (k + 1) * 32 + 4 * g);
        float4 r;
        r.x = ra * e.x * (bv.x * gk);
        r.y = ra * e.y * (bv.y * gk);
        r.z = ra * e.z * (bv.z * gk);
        r.w = ra * e.w * (bv.w * gk);
        __stcs(reinterpret_cast<float4*>(out + (size_t)k * 1024) + tid, r);
      }

    } else {
      for (int e = tid; e < Lc * m * m; e += kThreads) {
        const int k = e / (m * m), r = e - k * m * m, a = r / m, bb = r - a * m;
        const float gk = S.gh[k];
        out[e] = (S.al[k * 32 + a] * gk) * S.E[k * 1024 + swz(a, bb)] * (S.be[(k + 1) * 32 + bb] * gk);
      }
    }
  }
  return;

fallback:
  // exact log-space path for the whole instance, by the cluster's rank-0 CTA
  if (c != 0) return;
  __syncthreads();
  {
    float* sm = reinterpret_cast<float*>(smscan);
    small_pass(init, trans, T + 1, m, ws, logz, status, b, true, sm, n);
    __syncthreads();
    small_pass(init, trans, T + 1, m, ws, logz, status, b, false, sm, n);
    __syncthreads();
    marg_steps(init, trans, n, m, ws, logz, marg_init, marg_trans, b, 0, T, true);
    if (marg_trans)
      for (size_t e = (size_t)T * m * m + tid; e < (size_t)Tl * m * m; e += kThreads)
        marg_trans[(size_t)b * Tl * m * m + e] = 0.f;
  }
}

// Viterbi for m <= 32 (chain.py:98-114), one CTA per instance; theta tiles stream
// through a ring of kVD row-padded tiles (pitch 36), one 16-byte cp.async per thread
// per step; ONE CTA barrier per step publishes the new scores.
constexpr int kVD = 8;
constexpr int kVTP = 36;

__device__ __forceinline__ uint64_t dkey(double v) {
  const uint64_t u = (uint64_t)__double_as_longlong(v);
  return u ^ ((u >> 63) ? 0xffffffffffffffffull : 0x8000000000000000ull);
}
// lowest lane holding the maximum key (the reference's first argmax)
__device__ __forceinline__ int warp_argmax_key(uint64_t k) {
  const uint32_t hi = (uint32_t)(k >> 32), lo = (uint32_t)k;
  const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
  uint32_t cand = __ballot_sync(0xffffffffu, hi == mh);
  if (cand & (cand - 1)) {  // several equal high words: compare the low words
    const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    cand = __ballot_sync(0xffffffffu, hi == mh && lo == ml);
  }
  return __ffs(cand) - 1;
}

// Grouped Viterbi (m <= 32): kGP lanes per next tag, 256 threads.  Lane q of
// tag b's group scans the predecessors a = q, q + 8, q + 16, q + 24 with the
// reference's fp64 sums s_t[a] + theta_t[a][b] and a strict '>' (first maximum
// of its phase), then the group combines (value, a) pairs over three xor
// shuffles, ties to the lower a: the first maximum over all predecessors
// (chain.py:106).  With the tile pitch 36 the eight phases of four tags read
// 32 distinct banks.  (One warp per tag with a REDUX argmax: 49.4 vs 47.2 us at
// B=32 n=128; comparing on 64-bit integer keys instead of fp64: 55.4 us.)
constexpr int kGP = 8;
constexpr int kGT = 32 * kGP;

__global__ void __launch_bounds__(kGT, 1) chain_viterbi_grp_kernel(
    const float* __restrict__ init, const float* __restrict__ trans, int n, int m, int32_t* __restrict__ tags,
    double* __restrict__ score, int32_t* __restrict__ status, const int32_t* __restrict__ lengths) {
  extern __shared__ __align__(16) float smw[];
  float* ring = smw;                                                       // [kVD][32][kVTP]
  double* sv = reinterpret_cast<double*>(ring + kVD * 32 * kVTP);          // [2][32]
  uint8_t* back = reinterpret_cast<uint8_t*>(sv + 64);                     // [n][32]
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = tid / kGP, q = tid % kGP;  // next tag, predecessor phase
  const int nl = n, mm = m * m;  // nl: layout length; n: this instance's length (ragged batches)
  n = lengths ? min(max(lengths[b], 1), nl) : nl;
  const int T = n - 1;
  const float* th = trans + (size_t)b * (nl - 1) * mm;
  const bool full = (m == 32) && ((((uintptr_t)th) & 15) == 0);
  auto stage = [&](int t) {
    float* tile = ring + (t % kVD) * 32 * kVTP;
    if (full) {
      const int r = tid >> 3, c4 = (tid & 7) * 4;
      const unsigned dst = (unsigned)__cvta_generic_to_shared(tile + r * kVTP + c4);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(th + (size_t)t * 1024 + r * 32 + c4));
    } else {
      for (int e = tid; e < 1024; e += kGT) {
        const int r = e >> 5, c = e & 31;
        if (r < m && c < m) {
          const unsigned dst = (unsigned)__cvta_generic_to_shared(tile + r * kVTP + c);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(th + (size_t)t * mm + r * m + c));
        }
      }
    }
  };
  // tile t goes into ring slot t % kVD; the refill at step t is tile t + kVD - 1 into
  // the slot every thread finished reading at step t - 1 (behind this step's barrier)
  for (int d = 0; d < kVD - 1; ++d) {
    if (d < T) stage(d);
    cpa_commit();
  }
  int bad = 0;
  if (tid < 32) {
    const float x = tid < m ? init[(size_t)b * m + tid] : ninf();
    bad |= (tid < m) && bad_input(x);
    sv[tid] = tid < m ? (double)x : ninfd();
  }
  const bool live = nb < m;
  for (int t = 0; t < T; ++t) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kVD - 2));
    __syncthreads();  // tile t resident; s_t published; slot (t - 1) % kVD free
    const double* cur = sv + (t & 1) * 32;
    double* nxt = sv + ((t + 1) & 1) * 32;
    const float* col = ring + (t % kVD) * 32 * kVTP + nb;  // theta_t[a][nb] at col[a * kVTP]
    if (t + kVD - 1 < T) stage(t + kVD - 1);
    cpa_commit();
    double best = ninfd();
    int arg = q;
#pragma unroll
    for (int i = 0; i < 32 / kGP; ++i) {
      const int a = q + kGP * i;
      const float x = col[a * kVTP];
      const bool ok = live && a < m;
      bad |= ok && bad_input(x);
      const double v = ok ? cur[a] + (double)x : ninfd();
      if (v > best) { best = v; arg = a; }
    }
#pragma unroll
    for (int o = 1; o < kGP; o <<= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
      if (ob > best || (ob == best && oa < arg)) { best = ob; arg = oa; }
    }
    if (q == 0 && live) {
      nxt[nb] = best;
      back[(size_t)(t + 1) * 32 + nb] = (uint8_t)arg;
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  bad = __syncthreads_or(bad);  // also publishes the last scores
  if (warp == 0) {
    const bool alive = lane < m;
    const double* fin = sv + (T & 1) * 32;
    const double v = alive ? fin[lane] : ninfd();
    const int win = warp_argmax_key(dkey(v));  // final tag: first argmax (chain.py:111)
    const double bestf = __shfl_sync(0xffffffffu, v, win);
    int32_t* tg = tags + (size_t)b * nl;
    for (int t = n + lane; t < nl; t += 32) tg[t] = 0;  // past this instance's length
    if (lane == 0) {
      const bool vac = (bestf == ninfd());
      status[b] = bad ? SDB_ST_INVALID : (vac ? SDB_ST_VACUOUS : SDB_ST_OK);
      score[b] = bestf;
      int c = vac ? 0 : win;
      tg[n - 1] = c;
      for (int t = n - 2; t >= 0; --t) {
        c = vac ? 0 : back[(size_t)(t + 1) * 32 + c];
        tg[t] = c;
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

#ifdef SDB_SCAN_PROF
extern "C" int sdb_debug_scan_times(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, g_scan_t, bytes < sizeof(g_scan_t) ? bytes : sizeof(g_scan_t)) == cudaSuccess
             ? 0
             : -1;
}
#endif

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
  const int T = n - 1;
  if (m <= 32 && T >= 2 * kSC && (T + kSC - 1) / kSC <= kSLmax) {
    // time-parallel scan: one cluster of kSC CTAs per instance, one launch
    const size_t smem = scan_smem((T + kSC - 1) / kSC);
    auto kern = (m == 32) ? chain_scan_kernel<true> : chain_scan_kernel<false>;
    if (sdb_set_smem((const void*)kern, smem) != cudaSuccess)
      return SDB_ERR_CUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(B * kSC));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kSC;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, init, trans, n, m, ws, logz, marg_init, marg_trans, status,
                           (const int32_t*)nullptr) != cudaSuccess)
      return SDB_ERR_CUDA;
    SDB_CHECK_LAUNCH();
    return SDB_OK;
  }
  const bool lin = (m <= 32) && (n - 1 >= 2 * kLB);
  const size_t small_smem = (size_t)kD * m * m * 4 + (32 + 2 * kGroups * 32) * 4;
  if (lin) {
    const size_t smem = lin_smem_bytes();
    if (sdb_set_smem((const void*)chain_lin_kernel, smem) != cudaSuccess)
      return SDB_ERR_CUDA;
    chain_lin_kernel<<<(unsigned)(2 * B), kThreads, smem, s>>>(init, trans, n, m, ws, logz, status);
    SDB_CHECK_LAUNCH();
    // marginals of the linear instances (also merges the two passes' verdicts into ws.need)
    dim3 gl((unsigned)((n - 1 + kLinMargSteps - 1) / kLinMargSteps), (unsigned)B);
    chain_lin_marg_kernel<<<gl, kThreads, 0, s>>>(init, trans, n, m, ws, logz, marg_init, marg_trans);
    dim3 g((unsigned)((n - 1 + kStepsPerBlock - 1) / kStepsPerBlock), (unsigned)B);
    SDB_CHECK_LAUNCH();
    // exact log-space recomputation of the (rare) instances the linear path flagged
    if (sdb_set_smem((const void*)chain_fwd_bwd_small_kernel, small_smem) != cudaSuccess)
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
    if (sdb_set_smem((const void*)chain_fwd_bwd_small_kernel, small_smem) != cudaSuccess)
      return SDB_ERR_CUDA;
    chain_fwd_bwd_small_kernel<<<dim3((unsigned)B, 2), kThreads, small_smem, s>>>(init, trans, n, m, ws, logz,
                                                                                  status, 0);
  } else {
    size_t smem = (size_t)m * 4 * (1 + 2 * kGroups);
    if (smem > 48 * 1024) {
      if (sdb_set_smem((const void*)chain_fwd_bwd_kernel, smem) !=
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

// Ragged batches (per-instance lengths, no padding compute; chain.py:161-176 semantics
// without pad_chain): the arrays keep the batch layout of n positions, instance b uses
// its first lengths[b] (1 <= lengths[b] <= n); marginals / tags past it are 0.
// Served by the scan and Viterbi kernels: m <= 32, n <= kSC * kSLmax + 1.
extern "C" int sdb_chain_fb_lengths(const float* init, const float* trans, const int32_t* lengths, int64_t B,
                                    int32_t n, int32_t m, double* logz, float* marg_init, float* marg_trans,
                                    int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  if (B < 0 || n < 1 || m < 1 || !init || (n > 1 && !trans) || !lengths || !logz || !status) return SDB_ERR_ARG;
  if (m > 32 || (n - 1 + kSC - 1) / kSC > kSLmax) return SDB_ERR_UNSUPPORTED;
  if (B == 0) return SDB_OK;
  size_t need = 0;
  ChainWs ws = carve_chain(workspace, B, n, m, &need);
  if (!workspace || ws_bytes < need) return SDB_ERR_WORKSPACE;
  const int T = n - 1;
  const size_t smem = scan_smem((T + kSC - 1) / kSC);
  auto kern = (m == 32) ? chain_scan_kernel<true> : chain_scan_kernel<false>;
  if (sdb_set_smem((const void*)kern, smem) != cudaSuccess)
    return SDB_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(B * kSC));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kSC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, init, trans, n, m, ws, logz, marg_init, marg_trans, status, lengths) !=
      cudaSuccess)
    return SDB_ERR_CUDA;
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" int sdb_chain_viterbi_lengths(const float* init, const float* trans, const int32_t* lengths, int64_t B,
                                         int32_t n, int32_t m, int32_t* tags, double* score, int32_t* status,
                                         void* stream) {
  if (B < 0 || n < 1 || m < 1 || !init || (n > 1 && !trans) || !lengths || !tags || !score || !status)
    return SDB_ERR_ARG;
  const size_t smw = (size_t)kVD * 32 * kVTP * 4 + 64 * 8 + (size_t)n * 32 + 64;
  if (m > 32 || smw > 200 * 1024) return SDB_ERR_UNSUPPORTED;
  if (B == 0) return SDB_OK;
  if (sdb_set_smem((const void*)chain_viterbi_grp_kernel, smw) != cudaSuccess) return SDB_ERR_CUDA;
  chain_viterbi_grp_kernel<<<(unsigned)B, kGT, smw, (cudaStream_t)stream>>>(init, trans, n, m, tags, score, status,
                                                                            lengths);
  SDB_CHECK_LAUNCH();
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
    const size_t smw = (size_t)kVD * 32 * kVTP * 4 + 64 * 8 + (size_t)n * 32 + 64;  // ring, scores, backpointers
    if (smw <= 200 * 1024) {
      if (sdb_set_smem((const void*)chain_viterbi_grp_kernel, smw) != cudaSuccess) return SDB_ERR_CUDA;
      chain_viterbi_grp_kernel<<<(unsigned)B, kGT, smw, (cudaStream_t)stream>>>(init, trans, n, m, tags, score,
                                                                                status, nullptr);
      SDB_CHECK_LAUNCH();
      return SDB_OK;
    }
    const size_t smem = (size_t)(kD + 1) * m * kVP * 4 + 64 * 8 + (size_t)n * 32 + 64;
    if (smem <= 200 * 1024) {
      if (sdb_set_smem((const void*)chain_viterbi_small_kernel, smem) !=
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
    if (sdb_set_smem((const void*)chain_viterbi_kernel, smem) != cudaSuccess)
      return SDB_ERR_CUDA;
  }
  chain_viterbi_kernel<<<(unsigned)B, kThreads, smem, (cudaStream_t)stream>>>(
      init, trans, n, m, (uint16_t*)workspace, in_smem ? 1 : 0, tags, score, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
