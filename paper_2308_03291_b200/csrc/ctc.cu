// CTC over the blank-interleaved 2L+1 lattice: log-partition, per-frame
// vocabulary marginals, best expanded-state path.
//
// Reference: structdist alignment.py:231-336 (_expanded_labels,
// _ctc_predecessors, _ctc_forward, _ctc_backward, ctc_marginals, ctc_argmax,
// _ctc_walk).  Layout per instance: frame_potentials [T][V] fp32,
// targets [L] int32 (labels in 1..V-1), blank = 0.
//
// Schedule: one CTA per (instance, direction), frames in lockstep (one
// __syncthreads per frame).  Frame rows are prefetched kP frames ahead into a
// shared ring with cp.async and each state gathers its emission
// theta[t][lab(s)] from shared memory.
//   ctc_kernel<2>: fp64 max-plus alpha, a thread per state (S = 2L+1 <= 1024),
//            first-maximum back pointers and the walk (argmax).
//   ctc_dir_kernel<kMarg> (log Z: grid B x 1; marginals: grid B x 2): a thread
//            per (blank, label) state pair; the forward CTA stores alpha, the backward CTA beta, both as
//            fp32 offsets from per-(frame, warp) bases, concurrently; the
//            forward owns Z, the status and the label CSR.
//   ctc_marg_kernel: posteriors exp(alpha + beta - Z) reduced by label in a
//            fixed order (blank: lane-strided sums + butterfly; labels: the CSR
//            state list in increasing s), a warp per frame, streaming.
// Log values: fp64 in ctc_kernel (logZ, exact max-plus argmax); fp32 (value,
// integer offset) pairs in log2 units in ctc_dir_kernel, MUFU exp2/log2.
#include "common.cuh"

namespace {

constexpr int kP = 8;  // frame prefetch distance / ring depth

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

struct CtcSmem {
  double* a0;   // [S+2] ping (2 leading -inf pads)
  double* a1;   // [S+2] pong
  float* rows;  // [kP][V]
  int* lab;     // [S]
};

size_t ctc_smem_bytes(int S, int V, int L) {
  (void)L;
  return (size_t)2 * (S + 2) * 8 + (size_t)kP * V * 4 + (size_t)S * 4 + 128;
}

__device__ CtcSmem ctc_carve(char* p, int S, int V, int L) {
  (void)L;
  CtcSmem s;
  s.a0 = (double*)p; p += (size_t)(S + 2) * 8;
  s.a1 = (double*)p; p += (size_t)(S + 2) * 8;
  s.rows = (float*)p; p += (size_t)kP * V * 4;
  s.lab = (int*)p;
  return s;
}

__device__ __forceinline__ void load_row(const float* __restrict__ fp, int t, int V, float* dst) {
  for (int v = threadIdx.x; v < V; v += blockDim.x) cp_async4(dst + v, fp + (size_t)t * V + v);
}

template <int kMode>  // 2: max-plus path (log Z and marginals: ctc_dir_kernel)
__global__ void ctc_kernel(const float* __restrict__ fp_all, const int32_t* __restrict__ tg_all, int T, int V,
                           int L, int8_t* __restrict__ back_all, double* __restrict__ /*logz*/,
                           int32_t* __restrict__ path_all, double* __restrict__ score, int32_t* __restrict__ status) {
  static_assert(kMode == 2, "ctc_kernel modes");
  extern __shared__ __align__(16) char smraw[];
  const int S = 2 * L + 1;
  CtcSmem sm = ctc_carve(smraw, S, V, L);
  __shared__ int badsh;
  const int b = blockIdx.x, tid = threadIdx.x;
  const float* fp = fp_all + (size_t)b * T * V;
  const int32_t* tg = tg_all + (size_t)b * L;
  const int s = tid;
  const bool act = s < S;
  if (tid == 0) badsh = 0;
  __syncthreads();
  int mylab = 0;
  if (act) {
    mylab = (s & 1) ? tg[s >> 1] : 0;
    if ((s & 1) && (mylab < 1 || mylab >= V)) {
      atomicOr(&badsh, 1);
      mylab = 0;
    }
    sm.lab[s] = mylab;
  }
  __syncthreads();
  const bool skip = act && (s >= 2) && mylab != 0 && mylab != sm.lab[s - 2];
  // forward (alignment.py:248-269; max-plus with first-maximum back pointers, 304-318)
  double* prv = sm.a0 + 2;  // alpha[t-1]
  double* now = sm.a1 + 2;
  if (tid < 2) { sm.a0[tid] = ninfd(); sm.a1[tid] = ninfd(); }
  for (int k = 0; k < kP; ++k) {
    if (k < T) load_row(fp, k, V, sm.rows + (size_t)k * V);
    cp_commit();
  }
  int8_t* back = back_all + (size_t)b * T * S;
  int bad = 0;
  for (int t = 0; t < T; ++t) {
    cp_wait<kP - 1>();
    __syncthreads();
    const float* E = sm.rows + (size_t)(t % kP) * V;
    for (int v = tid; v < V; v += blockDim.x) bad |= bad_input(E[v]);
    double a = ninfd();
    if (act) {
      const double e = (double)E[mylab];
      if (t == 0) {
        a = (s <= 1) ? e : ninfd();
      } else {
        // first maximum in predecessor order [s, s-1, s-2] (alignment.py:239-245, 304-318)
        double best = prv[s];
        int k = 0;
        if (s >= 1 && prv[s - 1] > best) { best = prv[s - 1]; k = 1; }
        if (skip && prv[s - 2] > best) { best = prv[s - 2]; k = 2; }
        a = best + e;
        back[(size_t)t * S + s] = (int8_t)k;
      }
      now[s] = a;
    }
    __syncthreads();  // now[] complete; row t consumed
    {
      const int tn = t + kP;
      if (tn < T) load_row(fp, tn, V, sm.rows + (size_t)(tn % kP) * V);
      cp_commit();
    }
    double* tmp = prv; prv = now; now = tmp;
  }
  cp_wait<0>();
  if (bad) atomicOr(&badsh, 1);
  __syncthreads();
  // final states (alignment.py:263-264): [S-1] or [S-1, S-2]
  if (tid == 0) {
    const double f1 = prv[S - 1];
    const double f2 = (S > 1) ? prv[S - 2] : ninfd();
    double res = f1;
    int fin = S - 1;
    if (S > 1 && f2 > f1) { res = f2; fin = S - 2; }
    const int st = badsh ? SDB_ST_INVALID : (res == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
    status[b] = st;
    score[b] = res;
    int32_t* path = path_all + (size_t)b * T;
    int cs = fin;
    for (int t = T - 1; t >= 0; --t) {
      path[t] = (st == SDB_ST_OK) ? sm.lab[cs] : 0;
      if (t > 0 && st == SDB_ST_OK) cs -= back[(size_t)t * S + cs];
    }
  }
}

// log_partition + marginals as TWO independent CTAs per instance (grid B x 2):
// blockIdx.y = 0 runs the forward (alpha) over frames 0..T-1 and owns Z, the
// status and the label CSR; blockIdx.y = 1 runs the backward (beta) over
// T-1..0, concurrently.  The recursion is fp32 in log2 units carried as
// (v, O): value = v + O with O an integer-valued float re-chosen every frame
// (the alignment kernel's representation).  A state combines its three
// predecessors in the frame of the largest offset (exact integer
// differences), so no fp64 and no f32<->f64 conversion is on the per-frame
// chain; offsets stay exact while |value| < 2^24 (|log Z| < 1.1e7).  Dead
// (-inf) states carry O = kNoO, which is never the largest live offset.  Both
// directions store their vectors as fp32 offsets from the per-(frame, warp)
// maximum O; ctc_marg_kernel forms exp2(alpha + beta - Z).
constexpr float kNoO = -1.0e30f;

__device__ __forceinline__ float2 vo_dead() { return make_float2(ninf(), kNoO); }

// log2-sum-exp2 of two / three (v, O) terms plus e (log2 units), renormalised to
// |v| <= 1/2.  Branch-free on dead terms: a dead result has v = -inf and an
// offset <= kNoO (r, r2 clamp to kNoO, so offsets stay finite for any practical
// T), which is never the largest offset of a term with a live one.
__device__ __forceinline__ float2 vo_fin(float oref, float r, float v) {
  const float r2 = rintf(fmaxf(v, kNoO));
  return make_float2(v - r2, (oref + r) + r2);
}
__device__ __forceinline__ float2 vo_lse2(float2 x0, float2 x1, float e) {
  const float oref = fmaxf(x0.y, x1.y);
  const float t0 = x0.x + (x0.y - oref), t1 = x1.x + (x1.y - oref);
  const float r = rintf(fmaxf(fmaxf(t0, t1), kNoO));
  return vo_fin(oref, r, lg2(ex2(t0 - r) + ex2(t1 - r)) + e);
}
__device__ __forceinline__ float2 vo_lse3(float2 x0, float2 x1, float2 x2, float e) {
  const float oref = fmaxf(fmaxf(x0.y, x1.y), x2.y);
  const float t0 = x0.x + (x0.y - oref), t1 = x1.x + (x1.y - oref), t2 = x2.x + (x2.y - oref);
  const float r = rintf(fmaxf(fmaxf(fmaxf(t0, t1), t2), kNoO));
  return vo_fin(oref, r, lg2(ex2(t0 - r) + ex2(t1 - r) + ex2(t2 - r)) + e);
}
// (v, O) + e, renormalised
__device__ __forceinline__ float2 vo_add(float2 x, float e) { return vo_fin(x.y, 0.f, x.x + e); }

// Warp maximum of integer-valued offsets: clamped to >= -2^22 and shifted by
// 1.5 * 2^23, every offset is a positive float whose bit pattern orders like its
// value, so one unsigned REDUX finds the maximum.  Live offsets are exact above
// -2^22 (|log Z| < 2.9e6); dead ones clamp to the floor.
__device__ __forceinline__ float warp_max_off(float o) {
  constexpr float kMagic = 12582912.f;
  const uint32_t k = __float_as_uint(fmaxf(o, -4194304.f) + kMagic);
  return __uint_as_float(__reduce_max_sync(0xffffffffu, k)) - kMagic;
}

// Thread i owns the state pair (2i, 2i+1) -- blank 2i, label i -- for
// i = 0..L-1, and thread L-1 also owns the final blank 2L (L = 0: thread 0
// owns state 0), so S = 2L+1 <= 1024 takes L <= 512 threads.  A thread's
// previous values stay in registers; the one neighbour term crosses through
// shared memory: forward, alpha(2i-1) from thread i-1 (a blank has
// predecessors {2i, 2i-1}, a label {2i+1, 2i, 2i-1 if skip}); backward, c(2i+2),
// c(2i+3) from thread i+1 (a blank has successors {2i, 2i+1}, a label {2i+1,
// 2i+2, 2i+3 if skip}; the final blank only itself).  Workspace rows have the
// even pitch Sp = 2L+2 (one 8-byte store per pair), bases per 64-state warp.
size_t ctc_dir_smem_bytes(int S, int V, int L) {
  (void)S;
  return (size_t)3 * (L + 3) * 16 + (size_t)kP * V * 4 + (size_t)(2 * L + 1) * 4 + (size_t)(L + 1) * 4 +
         (size_t)(V + 1) * 4 + 128;
}
int ctc_dir_threads(int L) { return ((max(L, 1) + 31) / 32) * 32; }

// kMarg = false: the forward CTA alone (grid B x 1), no workspace -- the log-partition path
template <bool kMarg>
__global__ void ctc_dir_kernel(const float* __restrict__ fp_all, const int32_t* __restrict__ tg_all, int T, int V,
                               int L, float* __restrict__ wsa_all, float* __restrict__ wsabase_all,
                               float* __restrict__ wsb_all, float* __restrict__ wsbase_all,
                               int32_t* __restrict__ csr_all, double* __restrict__ logz,
                               int32_t* __restrict__ status) {
  extern __shared__ __align__(16) char smraw[];
  const int S = 2 * L + 1, Sp = 2 * L + 2;
  float4 *q0, *q1, *q2;  // three pair buffers [L+3] (one dead pad each side): one barrier per frame
  float* rows;
  int *lab, *lst, *off;
  {
    char* p = smraw;
    q0 = (float4*)p; p += (size_t)(L + 3) * 16;
    q1 = (float4*)p; p += (size_t)(L + 3) * 16;
    q2 = (float4*)p; p += (size_t)(L + 3) * 16;
    rows = (float*)p; p += (size_t)kP * V * 4;
    lab = (int*)p; p += (size_t)S * 4;
    lst = (int*)p; p += (size_t)(L + 1) * 4;
    off = (int*)p;
  }
  __shared__ int badsh;
  const int b = blockIdx.x, dir = blockIdx.y, tid = threadIdx.x, i = tid, lane = tid & 31, wq = tid >> 5;
  const bool act = i < max(L, 1), has1 = i < L, ext = (L >= 1) && (i == L - 1);
  const int ia = act ? i : 0;  // shared-memory neighbour reads of idle lanes stay in bounds
  const float* fp = fp_all + (size_t)b * T * V;
  const int32_t* tg = tg_all + (size_t)b * L;
  const float4 dead4 = make_float4(ninf(), kNoO, ninf(), kNoO);
  if (tid == 0) {
    badsh = 0;
    q0[0] = q1[0] = q2[0] = dead4;
    q0[L + 1] = q1[L + 1] = q2[L + 1] = dead4;
    q0[L + 2] = q1[L + 2] = q2[L + 2] = dead4;
  }
  int mylab = 0;  // label of state 2i+1
  if (has1) {
    mylab = tg[i];
    if (mylab < 1 || mylab >= V) {
      atomicOr(&badsh, 1);
      mylab = 0;
    }
  }
  if (act) {
    lab[2 * i] = 0;
    if (has1) lab[2 * i + 1] = mylab;
    if (ext) lab[2 * L] = 0;
  }
  __syncthreads();
  if (kMarg && dir == 0) {  // label CSR for ctc_marg_kernel: odd states by label, increasing s
    if (tid == 0) {
      for (int v = 0; v <= V; ++v) off[v] = 0;
      for (int k = 0; k < L; ++k) off[lab[2 * k + 1] + 1]++;
      for (int v = 0; v < V; ++v) off[v + 1] += off[v];
      for (int k = 0; k < L; ++k) lst[k] = -1;
      for (int k = 0; k < L; ++k) {
        int pos = off[lab[2 * k + 1]];
        while (lst[pos] >= 0) ++pos;
        lst[pos] = 2 * k + 1;
      }
    }
    __syncthreads();
    int32_t* csr = csr_all + (size_t)b * (V + 1 + L);
    for (int e = tid; e <= V; e += blockDim.x) csr[e] = off[e];
    for (int e = tid; e < L; e += blockDim.x) csr[V + 1 + e] = lst[e];
  }
  // a frame's states -> workspace: v + (O - base), base = the warp's largest offset (dead
  // states store -inf)
  auto store = [&](float* wrow, float* brow, float2 x0, float2 x1, float2 x2) {
    if constexpr (!kMarg) return;
    const float base = warp_max_off(act ? fmaxf(fmaxf(x0.y, x1.y), x2.y) : kNoO);
    if (act) *reinterpret_cast<float2*>(wrow + 2 * i) = make_float2(x0.x + (x0.y - base), x1.x + (x1.y - base));
    if (lane == 0) brow[wq] = base;
    if (ext) {
      wrow[2 * L] = x2.x + (x2.y - base);
      brow[L >> 5] = base;  // state 2L's 64-state group: this warp's, or (L % 32 == 0) an unused slot
    }
  };
  // Frames advance with ONE barrier each: the pair written at frame t goes to the buffer
  // last read at frame t-2 (every thread is past frame t-1 once it passes frame t's barrier),
  // and the row slot refilled after frame t's barrier is the one frame t-1 (forward) / t+1
  // (backward) consumed.
  if (kMarg && dir == 1) {
    // ======================= backward (alignment.py:272-287)
    float* wrow = wsb_all + (size_t)b * T * Sp + (size_t)(T - 1) * Sp;
    float* brow = wsbase_all + (size_t)b * T * 32 + (size_t)(T - 1) * 32;
    float4* cur = q0 + 1;  // c = beta[t+1] + theta[t+1][lab], per pair
    float4* nxt = q1 + 1;
    float4* spare = q2 + 1;
    for (int k = 0; k < kP; ++k) {
      const int t = T - 1 - k;
      if (t >= 0) load_row(fp, t, V, rows + (size_t)(t % kP) * V);
      cp_commit();
    }
    cp_wait<kP - 1>();
    __syncthreads();  // row T-1 landed
    // beta[T-1] = 0 on the final states 2L and 2L-1 (both thread L-1's; L = 0: thread 0's state 0)
    const bool f0 = (L == 0) && (i == 0);
    const float2 zero = make_float2(0.f, 0.f);
    float2 c0 = vo_dead(), c1 = vo_dead(), c2 = vo_dead();
    {
      const float* E = rows + (size_t)((T - 1) % kP) * V;
      if (f0) c0 = vo_add(zero, E[0] * SDB_LOG2E);
      if (ext) {
        c1 = vo_add(zero, E[mylab] * SDB_LOG2E);
        c2 = vo_add(zero, E[0] * SDB_LOG2E);
      }
      if (act) cur[i] = make_float4(c0.x, c0.y, c1.x, c1.y);
    }
    store(wrow, brow, f0 ? zero : vo_dead(), ext ? zero : vo_dead(), ext ? zero : vo_dead());
    const int lab3 = (i + 1 < L) ? tg[i + 1] : 0;  // label of state 2i+3
    const bool sk = (i + 1 < L) && lab3 != mylab;
    for (int t = T - 2; t >= 0; --t) {
      cp_wait<kP - 2>();
      __syncthreads();  // rows t+1 (consumed into cur) and t landed; cur complete
      {
        const int tn = t + 1 - kP;  // into row t+1's slot: no thread reads it any more
        if (tn >= 0) load_row(fp, tn, V, rows + (size_t)(tn % kP) * V);
        cp_commit();
      }
      wrow -= Sp;
      brow -= 32;
      const float* E = rows + (size_t)(t % kP) * V;
      const float eb = E[0] * SDB_LOG2E, el = E[mylab] * SDB_LOG2E;
      const float4 rn = cur[ia + 1];  // c(2i+2), c(2i+3) (dead pad past the end)
      const float2 s2 = ext ? c2 : make_float2(rn.x, rn.y);
      const float2 b0 = vo_lse2(c0, c1, 0.f);
      const float2 b1 = vo_lse3(c1, s2, sk ? make_float2(rn.z, rn.w) : vo_dead(), 0.f);
      const float2 b2 = c2;  // the final blank's only successor is itself
      c0 = vo_add(b0, eb);
      c1 = vo_add(b1, el);
      c2 = vo_add(b2, eb);
      if (act) nxt[i] = make_float4(c0.x, c0.y, c1.x, c1.y);
      store(wrow, brow, b0, b1, b2);
      float4* tmp = cur; cur = nxt; nxt = spare; spare = tmp;
    }
    cp_wait<0>();
    return;
  }
  // ======================= forward (alignment.py:248-269)
  float* wrow = wsa_all + (size_t)b * T * Sp;
  float* brow = wsabase_all + (size_t)b * T * 32;
  float4* prv = q0 + 1;
  float4* now = q1 + 1;
  float4* spare = q2 + 1;
  const int labm = (i >= 1 && has1) ? tg[i - 1] : 0;  // label of state 2i-1
  const bool skip = has1 && i >= 1 && labm != mylab;
  for (int k = 0; k < kP - 1; ++k) {
    if (k < T) load_row(fp, k, V, rows + (size_t)k * V);
    cp_commit();
  }
  int bad = 0;
  float2 a0 = vo_dead(), a1 = vo_dead(), a2 = vo_dead();
  for (int t = 0; t < T; ++t) {
    cp_wait<kP - 2>();
    __syncthreads();  // row t landed; alpha[t-1] complete; row t-1 consumed
    {
      const int tn = t + kP - 1;  // into row t-1's slot
      if (tn < T) load_row(fp, tn, V, rows + (size_t)(tn % kP) * V);
      cp_commit();
    }
    const float* E = rows + (size_t)(t % kP) * V;
    for (int v = tid; v < V; v += blockDim.x) bad |= bad_input(E[v]);
    const float eb = E[0] * SDB_LOG2E, el = E[mylab] * SDB_LOG2E;
    if (t == 0) {
      a0 = (i == 0) ? vo_add(make_float2(0.f, 0.f), eb) : vo_dead();
      a1 = (i == 0 && has1) ? vo_add(make_float2(0.f, 0.f), el) : vo_dead();
    } else {
      const float4 lf = prv[ia - 1];  // alpha(2i-2), alpha(2i-1) (dead pad before 0)
      const float2 am = make_float2(lf.z, lf.w);
      const float2 n0 = vo_lse2(a0, am, eb);
      const float2 n2 = vo_lse2(a2, a1, eb);  // the final blank 2L: {2L, 2L-1}
      a1 = vo_lse3(a1, a0, skip ? am : vo_dead(), el);
      a0 = n0;
      a2 = ext ? n2 : vo_dead();
      if (!has1) a1 = vo_dead();
    }
    if (act) now[i] = make_float4(a0.x, a0.y, a1.x, a1.y);
    if (ext) now[L] = make_float4(a2.x, a2.y, ninf(), kNoO);
    store(wrow, brow, a0, a1, a2);
    wrow += Sp;
    brow += 32;
    float4* tmp = prv; prv = now; now = spare; spare = tmp;
  }
  cp_wait<0>();
  if (bad) atomicOr(&badsh, 1);
  __syncthreads();
  if (tid == 0) {  // final states (alignment.py:263-264): 2L and 2L-1
    const float4 pl = (L >= 1) ? prv[L] : prv[0];
    const float2 f1 = make_float2(pl.x, pl.y);
    const float2 f2 = (L >= 1) ? make_float2(prv[L - 1].z, prv[L - 1].w) : vo_dead();
    const double d1 = (f1.x == ninf()) ? ninfd() : (double)f1.x + (double)f1.y;
    const double d2 = (f2.x == ninf()) ? ninfd() : (double)f2.x + (double)f2.y;
    const double M = fmax(d1, d2);
    const double Z2 = (M == ninfd()) ? ninfd() : M + log2(exp2(d1 - M) + exp2(d2 - M));
    const double Z = Z2 * (double)SDB_LN2;
    status[b] = badsh ? SDB_ST_INVALID : (Z == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
    logz[b] = Z;
  }
}

// Per-frame vocabulary marginals from the alpha/beta offsets ctc_dir_kernel left
// in the workspace (alignment.py:290-301): marg[t][v] = sum of post[t][s] over
// the states s with label v (blank: the L+1 even states; repeated labels
// accumulate), in increasing s -- a deterministic order.  Grid (frame blocks,
// instances), every frame independent, so this streams at HBM rate instead of
// sitting inside the sequential frame loop.
constexpr int kMargWarps = 8;       // warps per CTA, one frame per warp at a time
constexpr int kMargFrames = 32;     // frames per CTA (4 per warp)

// A warp owns whole frames: it stages the frame's posterior row in its own
// shared slice and reduces it with warp primitives only, so the warps of a CTA
// never wait on each other (the per-frame CTA barriers of a row-per-CTA layout
// left this kernel latency-bound).
// kVR > 0 (V <= 32 kVR): lane-owned labels v = lane + 32 k with their first two
// states cached in registers (the CSR fallback only for a label repeated three or
// more times); kVR = 0: every label through the CSR lists.
template <int kRowRegs, int kVR>  // kRowRegs >= ceil(S / 32): the row's states per lane
__global__ void __launch_bounds__(kMargWarps * 32) ctc_marg_kernel(
    const float* __restrict__ wsa_all, const float* __restrict__ wsabase_all, const float* __restrict__ wsb_all,
    const float* __restrict__ wsbase_all, const double* __restrict__ logz, const int32_t* __restrict__ csr_all,
    int T, int V, int L, const int32_t* __restrict__ status, float* __restrict__ marg_all) {
  extern __shared__ __align__(16) float cm[];
  const int S = 2 * L + 1;
  int* off = reinterpret_cast<int*>(cm);      // [V+1]
  int* lst = off + V + 1;                     // [L]
  float* prow_all = cm + ((V + 1 + L + 3) & ~3);  // [kMargWarps][S + 1]
  const int b = blockIdx.y, t0 = blockIdx.x * kMargFrames, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int t1 = min(t0 + kMargFrames, T);
  float* mg = marg_all + (size_t)b * T * V;
  if (status[b] != SDB_ST_OK) {  // vacuous / invalid: zero marginals (as the reference's -inf Z)
    for (int e = tid; e < (t1 - t0) * V; e += blockDim.x) mg[(size_t)t0 * V + e] = 0.f;
    return;
  }
  const int32_t* csr = csr_all + (size_t)b * (V + 1 + L);  // built by ctc_dir_kernel's forward CTA
  for (int e = tid; e <= V; e += blockDim.x) off[e] = csr[e];
  for (int e = tid; e < L; e += blockDim.x) lst[e] = csr[V + 1 + e];
  __syncthreads();
  // label v's states in increasing s: the first two in registers (-1: none), `many` beyond
  int s1[kVR > 0 ? kVR : 1], s2[kVR > 0 ? kVR : 1];
  bool many[kVR > 0 ? kVR : 1];
#pragma unroll
  for (int k = 0; k < kVR; ++k) {
    const int v = lane + 32 * k;
    const int o0 = (v >= 1 && v < V) ? off[v] : 0, o1 = (v >= 1 && v < V) ? off[v + 1] : 0;
    s1[k] = (o1 > o0) ? lst[o0] : -1;
    s2[k] = (o1 > o0 + 1) ? lst[o0 + 1] : -1;
    many[k] = o1 > o0 + 2;
  }
  float* prow = prow_all + (size_t)warp * (S + 1);  // even slice pitch: float2 stores
  const int Sp = S + 1;  // ctc_dir_kernel's even row pitch
  const float* pa = wsa_all + (size_t)b * T * Sp;
  const float* pb = wsb_all + (size_t)b * T * Sp;
  const float* ba = wsabase_all + (size_t)b * T * 32;
  const float* bb = wsbase_all + (size_t)b * T * 32;
  const double Z2 = logz[b] * 1.4426950408889634;  // offsets and bases are log2 units
  // the warp's next frame is loaded into registers while the current one is reduced: lane l
  // holds the (blank, label) state pairs j = l + 32 u of both offset rows as float2 (the
  // direction kernel's pair layout); pair j's base group is j >> 5 = u.  Lane g loads the two
  // bases of group g and forms their fp64 combination with Z once; the pair loop shuffles it.
  constexpr int kPR = (kRowRegs + 1) / 2;  // pairs per lane
  float2 xa[kPR], xb[kPR];
  float ca, cb;
  auto fetch = [&](int t) {
    const float2* sa = reinterpret_cast<const float2*>(pa + (size_t)t * Sp);
    const float2* sb = reinterpret_cast<const float2*>(pb + (size_t)t * Sp);
#pragma unroll
    for (int u = 0; u < kPR; ++u) {
      const int j = lane + 32 * u;
      if (j <= L) {
        xa[u] = sa[j];
        xb[u] = sb[j];
      }
    }
    ca = ba[(size_t)t * 32 + lane];
    cb = bb[(size_t)t * 32 + lane];
  };
  if (t0 + warp < t1) fetch(t0 + warp);
  for (int t = t0 + warp; t < t1; t += kMargWarps) {
    const float cl = (float)((double)ca + (double)cb - Z2);  // base group `lane` (>= ceil((L+1)/32) unused)
    float bl = 0.f;  // blank: the even state of every pair
#pragma unroll
    for (int u = 0; u < kPR; ++u) {
      const int j = lane + 32 * u;
      const float c = __shfl_sync(0xffffffffu, cl, u);
      if (j <= L) {
        // an -inf offset gives ex2(-inf) = +0 (no +inf offsets); state 2L+1 does not exist
        const float p0 = ex2(c + xa[u].x + xb[u].x);
        const float p1 = (j < L) ? ex2(c + xa[u].y + xb[u].y) : 0.f;
        *reinterpret_cast<float2*>(prow + 2 * j) = make_float2(p0, p1);
        bl += p0;
      }
    }
    if (t + kMargWarps < t1) fetch(t + kMargWarps);
    bl = warp_sum(bl);
    __syncwarp();
    float* mrow = mg + (size_t)t * V;
    if constexpr (kVR > 0) {
#pragma unroll
      for (int k = 0; k < kVR; ++k) {
        const int v = lane + 32 * k;
        if (v < V) {
          float acc = 0.f;
          if (s1[k] >= 0) acc += prow[s1[k]];
          if (s2[k] >= 0) acc += prow[s2[k]];
          if (many[k])
            for (int q = off[v] + 2; q < off[v + 1]; ++q) acc += prow[lst[q]];
          mrow[v] = (v == 0) ? bl : acc;
        }
      }
    } else {
      for (int v = lane; v < V; v += 32) {
        float acc = 0.f;
        if (v == 0) {
          acc = bl;
        } else {
          for (int q = off[v]; q < off[v + 1]; ++q) acc += prow[lst[q]];
        }
        mrow[v] = acc;
      }
    }
    __syncwarp();  // the slice is rewritten for the warp's next frame
  }
}

struct CtcWs {
  float* wsa;      // [B][T][S+1] alpha offsets
  float* wsabase;  // [B][T][32] per-warp (64-state) alpha bases
  float* wsb;      // [B][T][S+1] beta offsets
  float* wsbase;   // [B][T][32] per-warp (64-state) beta bases
  int32_t* csr;    // [B][V+1+L] label CSR (offsets, odd states by label)
  int8_t* back;
};

CtcWs ctc_carve_ws(void* base, int64_t B, int T, int V, int L, int mode, size_t* bytes) {
  const int S = 2 * L + 1;
  Carve c(base);
  CtcWs w{};
  if (mode == 1) {
    w.wsa = c.take<float>((size_t)B * T * (S + 1));
    w.wsabase = c.take<float>((size_t)B * T * 32);
    w.wsb = c.take<float>((size_t)B * T * (S + 1));
    w.wsbase = c.take<float>((size_t)B * T * 32);
    w.csr = c.take<int32_t>((size_t)B * (V + 1 + L));
  }
  if (mode == 2) w.back = c.take<int8_t>((size_t)B * T * S);
  *bytes = c.used;
  return w;
}

bool ctc_fast_ok(int V, int L) {
  const int S = 2 * L + 1;
  return S <= 1024 && ctc_smem_bytes(S, V, L) <= 200 * 1024 && ctc_dir_smem_bytes(S, V, L) <= 200 * 1024;
}

}  // namespace

// ctc_gen.cu: states strided over the threads, fp64, for larger lattices
bool ctc_gen_ok(int L);
size_t ctc_gen_workspace(int64_t B, int T, int L, int mode);
int ctc_gen_launch(int mode, const float* fp, const int32_t* tg, int64_t B, int T, int V, int L, void* ws,
                   size_t ws_bytes, double* out, float* marg, int32_t* path, int32_t* status, cudaStream_t s);

namespace {
int ctc_check(int64_t B, int T, int V, int L) {
  if (B < 0 || T < 1 || V < 1 || L < 0) return SDB_ERR_ARG;
  if (!ctc_fast_ok(V, L) && !ctc_gen_ok(L)) return SDB_ERR_UNSUPPORTED;
  return SDB_OK;
}

template <int kMode>
int ctc_launch(const float* fp, const int32_t* tg, int64_t B, int T, int V, int L, CtcWs ws, double* logz,
               float* marg, int32_t* path, double* score, int32_t* status, cudaStream_t s) {
  const int S = 2 * L + 1;
  const int threads = ((S + 31) / 32) * 32;
  if constexpr (kMode == 0) {  // log Z: the forward direction of the marginal kernel
    const size_t dsmem = ctc_dir_smem_bytes(S, V, L);
    if (dsmem > 48 * 1024 && sdb_set_smem((const void*)ctc_dir_kernel<false>, dsmem) != cudaSuccess)
      return SDB_ERR_CUDA;
    ctc_dir_kernel<false><<<dim3((unsigned)B, 1), ctc_dir_threads(L), dsmem, s>>>(
        fp, tg, T, V, L, nullptr, nullptr, nullptr, nullptr, nullptr, logz, status);
  } else if constexpr (kMode == 1) {
    const size_t dsmem = ctc_dir_smem_bytes(S, V, L);
    if (dsmem > 48 * 1024 &&
        sdb_set_smem((const void*)ctc_dir_kernel<true>, dsmem) != cudaSuccess)
      return SDB_ERR_CUDA;
    ctc_dir_kernel<true><<<dim3((unsigned)B, 2), ctc_dir_threads(L), dsmem, s>>>(fp, tg, T, V, L, ws.wsa, ws.wsabase, ws.wsb,
                                                                ws.wsbase, ws.csr, logz, status);
  } else {
    const size_t smem = ctc_smem_bytes(S, V, L);
    if (sdb_set_smem((const void*)ctc_kernel<kMode>, smem) != cudaSuccess)
      return SDB_ERR_CUDA;
    ctc_kernel<kMode><<<(unsigned)B, threads, smem, s>>>(fp, tg, T, V, L, ws.back, logz, path, score, status);
  }
  SDB_CHECK_LAUNCH();
  if (kMode == 1) {
    const int S2 = 2 * L + 1;
    const size_t msmem = (((size_t)(V + 1 + L) + 3) & ~(size_t)3) * 4 + (size_t)kMargWarps * (S2 + 1) * 4;
    dim3 g((unsigned)((T + kMargFrames - 1) / kMargFrames), (unsigned)B);
    const int rr = (S2 + 31) / 32;
    const bool vr = V <= 128;
    const void* kf = rr <= 9 ? (vr ? (const void*)ctc_marg_kernel<9, 4> : (const void*)ctc_marg_kernel<9, 0>)
                             : (vr ? (const void*)ctc_marg_kernel<32, 4> : (const void*)ctc_marg_kernel<32, 0>);
    if (msmem > 48 * 1024 && sdb_set_smem(kf, msmem) != cudaSuccess) return SDB_ERR_CUDA;
    if (rr <= 9 && vr)
      ctc_marg_kernel<9, 4><<<g, kMargWarps * 32, msmem, s>>>(ws.wsa, ws.wsabase, ws.wsb, ws.wsbase, logz, ws.csr, T,
                                                             V, L, status, marg);
    else if (rr <= 9)
      ctc_marg_kernel<9, 0><<<g, kMargWarps * 32, msmem, s>>>(ws.wsa, ws.wsabase, ws.wsb, ws.wsbase, logz, ws.csr, T,
                                                             V, L, status, marg);
    else if (vr)
      ctc_marg_kernel<32, 4><<<g, kMargWarps * 32, msmem, s>>>(ws.wsa, ws.wsabase, ws.wsb, ws.wsbase, logz, ws.csr,
                                                              T, V, L, status, marg);
    else
      ctc_marg_kernel<32, 0><<<g, kMargWarps * 32, msmem, s>>>(ws.wsa, ws.wsabase, ws.wsb, ws.wsbase, logz, ws.csr,
                                                              T, V, L, status, marg);
    SDB_CHECK_LAUNCH();
  }
  return SDB_OK;
}

}  // namespace

extern "C" size_t sdb_ctc_fb_workspace(int64_t B, int32_t T, int32_t V, int32_t L) {
  if (!ctc_fast_ok(V, L)) return ctc_gen_workspace(B, T, L, 1);
  size_t bytes = 0;
  ctc_carve_ws(nullptr, B, T, V, L, 1, &bytes);
  return bytes;
}

extern "C" int sdb_ctc_fb(const float* frame_potentials, const int32_t* targets, int64_t B, int32_t T, int32_t V,
                          int32_t L, double* logz, float* marg, int32_t* status, void* workspace, size_t ws_bytes,
                          void* stream) {
  int rc = ctc_check(B, T, V, L);
  if (rc) return rc;
  if (!frame_potentials || (L > 0 && !targets) || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (!ctc_fast_ok(V, L))
    return ctc_gen_launch(marg ? 1 : 0, frame_potentials, targets, B, T, V, L, workspace, ws_bytes, logz, marg,
                          nullptr, status, s);
  if (!marg) return ctc_launch<0>(frame_potentials, targets, B, T, V, L, CtcWs{}, logz, nullptr, nullptr, nullptr, status, s);
  size_t need = 0;
  CtcWs ws = ctc_carve_ws(workspace, B, T, V, L, 1, &need);
  if (!workspace || ws_bytes < need) return SDB_ERR_WORKSPACE;
  return ctc_launch<1>(frame_potentials, targets, B, T, V, L, ws, logz, marg, nullptr, nullptr, status, s);
}

extern "C" size_t sdb_ctc_viterbi_workspace(int64_t B, int32_t T, int32_t V, int32_t L) {
  if (!ctc_fast_ok(V, L)) return ctc_gen_workspace(B, T, L, 2);
  size_t bytes = 0;
  ctc_carve_ws(nullptr, B, T, V, L, 2, &bytes);
  return bytes;
}

extern "C" int sdb_ctc_viterbi(const float* frame_potentials, const int32_t* targets, int64_t B, int32_t T,
                               int32_t V, int32_t L, int32_t* labels, double* score, int32_t* status,
                               void* workspace, size_t ws_bytes, void* stream) {
  int rc = ctc_check(B, T, V, L);
  if (rc) return rc;
  if (!frame_potentials || (L > 0 && !targets) || !labels || !score || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!ctc_fast_ok(V, L))
    return ctc_gen_launch(2, frame_potentials, targets, B, T, V, L, workspace, ws_bytes, score, nullptr, labels,
                          status, (cudaStream_t)stream);
  size_t need = 0;
  CtcWs ws = ctc_carve_ws(workspace, B, T, V, L, 2, &need);
  if (!workspace || ws_bytes < need) return SDB_ERR_WORKSPACE;
  return ctc_launch<2>(frame_potentials, targets, B, T, V, L, ws, nullptr, nullptr, labels, score, status,
                       (cudaStream_t)stream);
}
