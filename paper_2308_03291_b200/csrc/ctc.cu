// CTC over the blank-interleaved 2L+1 lattice: log-partition, per-frame
// vocabulary marginals, best expanded-state path.
//
// Reference: structdist alignment.py:231-336 (_expanded_labels,
// _ctc_predecessors, _ctc_forward, _ctc_backward, ctc_marginals, ctc_argmax,
// _ctc_walk).  Layout per instance: frame_potentials [T][V] fp32,
// targets [L] int32 (labels in 1..V-1), blank = 0.
//
// Schedule: one CTA per (instance, direction), one thread per lattice state s
// (S = 2L+1 <= 1024), frames in lockstep (one __syncthreads per frame).  Frame
// rows are prefetched kP frames ahead into a shared ring with cp.async and each
// state gathers its emission theta[t][lab(s)] from shared memory.
//   ctc_kernel<0/2>: alpha (log-sum-exp) or the max-plus alpha with
//            first-maximum back pointers and the walk (logZ, argmax).
//   ctc_dir_kernel (marginals, grid B x 2): the forward CTA stores alpha, the
//            backward CTA beta, both as fp32 offsets from per-(frame, warp)
//            bases, concurrently; the forward owns Z, the status and the label
//            CSR.
//   ctc_marg_kernel: posteriors exp(alpha + beta - Z) reduced by label in a
//            fixed order (blank: lane-strided sums + butterfly; labels: the CSR
//            state list in increasing s), a warp per frame, streaming.
// Log values are fp64 on the recursion; exp/log fp32 MUFU on differences.
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

template <int kMode>  // 0 logZ only, 2 max-plus path (marginals: ctc_dir_kernel)
__global__ void ctc_kernel(const float* __restrict__ fp_all, const int32_t* __restrict__ tg_all, int T, int V,
                           int L, int8_t* __restrict__ back_all, double* __restrict__ logz,
                           int32_t* __restrict__ path_all, double* __restrict__ score, int32_t* __restrict__ status) {
  static_assert(kMode == 0 || kMode == 2, "ctc_kernel modes");
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
  int8_t* back = (kMode == 2) ? back_all + (size_t)b * T * S : nullptr;
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
      } else if (kMode == 2) {
        // first maximum in predecessor order [s, s-1, s-2] (alignment.py:239-245, 304-318)
        double best = prv[s];
        int k = 0;
        if (s >= 1 && prv[s - 1] > best) { best = prv[s - 1]; k = 1; }
        if (skip && prv[s - 2] > best) { best = prv[s - 2]; k = 2; }
        a = best + e;
        back[(size_t)t * S + s] = (int8_t)k;
      } else {
        const double x0 = prv[s], x1 = prv[s - 1], x2 = skip ? prv[s - 2] : ninfd();
        const double M = fmax(fmax(x0, x1), x2);
        if (M != ninfd()) {
          const float sum = fexp((float)(x0 - M)) + fexp((float)(x1 - M)) + fexp((float)(x2 - M));
          a = M + (double)flog(sum) + e;
        }
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
    double res;
    int fin = S - 1;
    if (kMode == 2) {
      res = f1;
      if (S > 1 && f2 > f1) { res = f2; fin = S - 2; }
    } else {
      const double M = fmax(f1, f2);
      res = (M == ninfd()) ? ninfd() : M + (double)flog(fexp((float)(f1 - M)) + fexp((float)(f2 - M)));
    }
    const int st = badsh ? SDB_ST_INVALID : (res == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
    status[b] = st;
    if (kMode == 2) {
      score[b] = res;
      int32_t* path = path_all + (size_t)b * T;
      int cs = fin;
      for (int t = T - 1; t >= 0; --t) {
        path[t] = (st == SDB_ST_OK) ? sm.lab[cs] : 0;
        if (t > 0 && st == SDB_ST_OK) cs -= back[(size_t)t * S + cs];
      }
    } else {
      logz[b] = res;
    }
  }
}

// log_partition + marginals as TWO independent CTAs per instance (grid B x 2):
// blockIdx.y = 0 runs the forward (alpha) over frames 0..T-1 and owns Z, the
// status and the label CSR; blockIdx.y = 1 runs the backward (beta) over
// T-1..0.  Both store their vectors as fp32 offsets from a per-(frame, warp)
// fp64 base; ctc_marg_kernel forms exp(alpha + beta - Z).  Twice the CTAs of
// one fwd-then-bwd CTA per instance, and each runs half the frames: the
// per-frame latency chains of the two directions overlap across the SM
// instead of running back to back.
size_t ctc_dir_smem_bytes(int S, int V, int L) {
  return (size_t)3 * (S + 2) * 8 + (size_t)kP * V * 4 + (size_t)S * 4 + (size_t)(L + 1) * 4 + (size_t)(V + 1) * 4 +
         128;
}

__global__ void ctc_dir_kernel(const float* __restrict__ fp_all, const int32_t* __restrict__ tg_all, int T, int V,
                               int L, float* __restrict__ wsa_all, float* __restrict__ wsabase_all,
                               float* __restrict__ wsb_all, float* __restrict__ wsbase_all,
                               int32_t* __restrict__ csr_all, double* __restrict__ logz,
                               int32_t* __restrict__ status) {
  extern __shared__ __align__(16) char smraw[];
  const int S = 2 * L + 1;
  double *a0, *a1, *a2;  // three vector buffers: one barrier per frame
  float* rows;
  int *lab, *lst, *off;
  {
    char* p = smraw;
    a0 = (double*)p; p += (size_t)(S + 2) * 8;
    a1 = (double*)p; p += (size_t)(S + 2) * 8;
    a2 = (double*)p; p += (size_t)(S + 2) * 8;
    rows = (float*)p; p += (size_t)kP * V * 4;
    lab = (int*)p; p += (size_t)S * 4;
    lst = (int*)p; p += (size_t)(L + 1) * 4;
    off = (int*)p;
  }
  __shared__ int badsh;
  const int b = blockIdx.x, dir = blockIdx.y, tid = threadIdx.x, s = tid, lane = tid & 31, wq = tid >> 5;
  const bool act = s < S;
  const float* fp = fp_all + (size_t)b * T * V;
  const int32_t* tg = tg_all + (size_t)b * L;
  if (tid == 0) badsh = 0;
  __syncthreads();
  int mylab = 0;
  if (act) {
    mylab = (s & 1) ? tg[s >> 1] : 0;
    if ((s & 1) && (mylab < 1 || mylab >= V)) {
      atomicOr(&badsh, 1);
      mylab = 0;
    }
    lab[s] = mylab;
  }
  __syncthreads();
  if (dir == 0) {  // label CSR for ctc_marg_kernel: odd states by label, increasing s
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
  // vectors as fp32 offsets from a per-warp base (one REDUX max per frame, no CTA reduction).
  // The base is the warp maximum truncated to its high word (20 mantissa bits), found by a REDUX
  // on the high words' order-preserving keys: a double that is exactly an fp32 value, so it is
  // stored as one, and one f64->f32 conversion per state (the offset) is all the store costs.
  auto store = [&](float* ws, float* wsbase, int t, double v) {
    const double bm = warp_max_hi(v);
    const double base = (bm == ninfd()) ? 0.0 : bm;
    if (act) ws[(size_t)t * S + s] = (v == ninfd()) ? ninf() : (float)(v - base);
    if (lane == 0) wsbase[(size_t)t * 32 + wq] = (float)base;
  };
  if (tid < 2) { a0[tid] = ninfd(); a1[tid] = ninfd(); a2[tid] = ninfd(); }
  // Frames advance with ONE barrier each: the vector written at frame t goes to the buffer
  // last read at frame t-2 (every thread is past frame t-1 once it passes frame t's barrier),
  // and the row slot refilled after frame t's barrier is the one frame t-1 (forward) / t+1
  // (backward) consumed.
  if (dir == 1) {
    // ======================= backward (alignment.py:272-287)
    float* wsb = wsb_all + (size_t)b * T * S;
    float* wsbase = wsbase_all + (size_t)b * T * 32;
    double* cur = a0 + 2;  // beta[t+1][*] + theta[t+1][lab(*)]
    double* nxt = a1 + 2;
    double* spare = a2 + 2;
    for (int k = 0; k < kP; ++k) {
      const int t = T - 1 - k;
      if (t >= 0) load_row(fp, t, V, rows + (size_t)(t % kP) * V);
      cp_commit();
    }
    // the ring holds beta[t+1][s] + theta[t+1][lab(s)] (the successor term every predecessor of
    // s reads), so a state converts and adds ONE emission per frame instead of three
    cp_wait<kP - 1>();
    __syncthreads();  // row T-1 landed
    if (act) {
      const double b0 = (s == S - 1 || s == S - 2) ? 0.0 : ninfd();
      cur[s] = b0 + (double)rows[(size_t)((T - 1) % kP) * V + mylab];
    }
    store(wsb, wsbase, T - 1, (act && (s == S - 1 || s == S - 2)) ? 0.0 : ninfd());
    const bool has1 = act && (s + 1 < S);
    const int lab2 = (act && s + 2 < S) ? lab[s + 2] : 0;
    const bool sk2 = act && (s + 2 < S) && lab2 != 0 && lab2 != mylab;
    for (int t = T - 2; t >= 0; --t) {
      cp_wait<kP - 2>();
      __syncthreads();  // rows t+1 (consumed into cur) and t landed; cur complete
      {
        const int tn = t + 1 - kP;  // into row t+1's slot: no thread reads it any more
        if (tn >= 0) load_row(fp, tn, V, rows + (size_t)(tn % kP) * V);
        cp_commit();
      }
      const float* E = rows + (size_t)(t % kP) * V;
      double v = ninfd();
      if (act) {
        const double x0 = cur[s];
        const double x1 = has1 ? cur[s + 1] : ninfd();
        const double x2 = sk2 ? cur[s + 2] : ninfd();
        const double M = fmax(fmax(x0, x1), x2);
        if (M != ninfd()) {
          const float e = fexp((float)(x0 - M)) + fexp((float)(x1 - M)) + fexp((float)(x2 - M));
          v = M + (double)flog(e);
        }
        nxt[s] = v + (double)E[mylab];
      }
      store(wsb, wsbase, t, v);
      double* tmp = cur; cur = nxt; nxt = spare; spare = tmp;
    }
    cp_wait<0>();
    return;
  }
  // ======================= forward (alignment.py:248-269)
  float* wsa = wsa_all + (size_t)b * T * S;
  float* wsabase = wsabase_all + (size_t)b * T * 32;
  double* prv = a0 + 2;
  double* now = a1 + 2;
  double* spare = a2 + 2;
  const bool skip = act && (s >= 2) && mylab != 0 && mylab != lab[s - 2];
  for (int k = 0; k < kP - 1; ++k) {
    if (k < T) load_row(fp, k, V, rows + (size_t)k * V);
    cp_commit();
  }
  int bad = 0;
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
    double a = ninfd();
    if (act) {
      const double e = (double)E[mylab];
      if (t == 0) {
        a = (s <= 1) ? e : ninfd();
      } else {
        const double x0 = prv[s], x1 = prv[s - 1], x2 = skip ? prv[s - 2] : ninfd();
        const double M = fmax(fmax(x0, x1), x2);
        if (M != ninfd()) {
          const float sum = fexp((float)(x0 - M)) + fexp((float)(x1 - M)) + fexp((float)(x2 - M));
          a = M + (double)flog(sum) + e;
        }
      }
      now[s] = a;
    }
    store(wsa, wsabase, t, a);
    double* tmp = prv; prv = now; now = spare; spare = tmp;
  }
  cp_wait<0>();
  if (bad) atomicOr(&badsh, 1);
  __syncthreads();
  if (tid == 0) {  // final states (alignment.py:263-264): [S-1] or [S-1, S-2]
    const double f1 = prv[S - 1];
    const double f2 = (S > 1) ? prv[S - 2] : ninfd();
    const double M = fmax(f1, f2);
    const double Z = (M == ninfd()) ? ninfd() : M + (double)flog(fexp((float)(f1 - M)) + fexp((float)(f2 - M)));
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
template <int kRowRegs>  // >= ceil(S / 32): the row's states per lane
__global__ void __launch_bounds__(kMargWarps * 32) ctc_marg_kernel(
    const float* __restrict__ wsa_all, const float* __restrict__ wsabase_all, const float* __restrict__ wsb_all,
    const float* __restrict__ wsbase_all, const double* __restrict__ logz, const int32_t* __restrict__ csr_all,
    int T, int V, int L, const int32_t* __restrict__ status, float* __restrict__ marg_all) {
  extern __shared__ __align__(16) float cm[];
  const int S = 2 * L + 1;
  int* off = reinterpret_cast<int*>(cm);      // [V+1]
  int* lst = off + V + 1;                     // [L]
  float* prow_all = cm + ((V + 1 + L + 3) & ~3);  // [kMargWarps][S]
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
  float* prow = prow_all + (size_t)warp * S;
  const float* pa = wsa_all + (size_t)b * T * S;
  const float* pb = wsb_all + (size_t)b * T * S;
  const float* ba = wsabase_all + (size_t)b * T * 32;
  const float* bb = wsbase_all + (size_t)b * T * 32;
  const double Z = logz[b];
  // the warp's next frame (both offsets and the two bases of each 32-state group) is loaded into
  // registers while the current one is reduced; the posterior of state e = 32 u + lane is
  // exp(alpha + beta - Z): bases and Z combined in fp64, the offsets added in fp32
  // Lane g loads the two bases of 32-state group g (one coalesced load each) and forms that
  // group's fp64 combination once; the state loop takes it by shuffle.
  float xa[kRowRegs], xb[kRowRegs], ca, cb;
  auto fetch = [&](int t) {
    const float* sa = pa + (size_t)t * S;
    const float* sb = pb + (size_t)t * S;
#pragma unroll
    for (int u = 0; u < kRowRegs; ++u) {
      const int e = lane + 32 * u;
      if (e < S) {
        xa[u] = sa[e];
        xb[u] = sb[e];
      }
    }
    ca = ba[(size_t)t * 32 + lane];
    cb = bb[(size_t)t * 32 + lane];
  };
  if (t0 + warp < t1) fetch(t0 + warp);
  for (int t = t0 + warp; t < t1; t += kMargWarps) {
    const float cl = (float)((double)ca + (double)cb - Z);  // group `lane` (groups >= ceil(S/32) unused)
#pragma unroll
    for (int u = 0; u < kRowRegs; ++u) {
      const int e = lane + 32 * u;
      const float c = __shfl_sync(0xffffffffu, cl, u);
      if (e < S) {
        prow[e] = fexp(c + xa[u] + xb[u]);  // an -inf offset gives ex2(-inf) = +0 (no +inf offsets)
      }
    }
    if (t + kMargWarps < t1) fetch(t + kMargWarps);
    __syncwarp();
    // blank: the even states, fixed order (lane-strided partial sums, then a butterfly)
    float bl = 0.f;
    for (int e = 2 * lane; e < S; e += 64) bl += prow[e];
    bl = warp_sum(bl);
    for (int v = lane; v < V; v += 32) {
      float acc = 0.f;
      if (v == 0) {
        acc = bl;
      } else {
        for (int q = off[v]; q < off[v + 1]; ++q) acc += prow[lst[q]];
      }
      mg[(size_t)t * V + v] = acc;
    }
    __syncwarp();  // the slice is rewritten for the warp's next frame
  }
}

struct CtcWs {
  float* wsa;      // [B][T][S] alpha offsets
  float* wsabase;  // [B][T][32] per-warp alpha bases
  float* wsb;      // [B][T][S] beta offsets
  float* wsbase;   // [B][T][32] per-warp beta bases
  int32_t* csr;    // [B][V+1+L] label CSR (offsets, odd states by label)
  int8_t* back;
};

CtcWs ctc_carve_ws(void* base, int64_t B, int T, int V, int L, int mode, size_t* bytes) {
  const int S = 2 * L + 1;
  Carve c(base);
  CtcWs w{};
  if (mode == 1) {
    w.wsa = c.take<float>((size_t)B * T * S);
    w.wsabase = c.take<float>((size_t)B * T * 32);
    w.wsb = c.take<float>((size_t)B * T * S);
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
  if constexpr (kMode == 1) {
    const size_t dsmem = ctc_dir_smem_bytes(S, V, L);
    if (dsmem > 48 * 1024 &&
        sdb_set_smem((const void*)ctc_dir_kernel, dsmem) != cudaSuccess)
      return SDB_ERR_CUDA;
    ctc_dir_kernel<<<dim3((unsigned)B, 2), threads, dsmem, s>>>(fp, tg, T, V, L, ws.wsa, ws.wsabase, ws.wsb,
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
    const size_t msmem = (((size_t)(V + 1 + L) + 3) & ~(size_t)3) * 4 + (size_t)kMargWarps * S2 * 4;
    dim3 g((unsigned)((T + kMargFrames - 1) / kMargFrames), (unsigned)B);
    const int rr = (S2 + 31) / 32;
    if (rr <= 9) {
      if (msmem > 48 * 1024 && sdb_set_smem((const void*)ctc_marg_kernel<9>, msmem) != cudaSuccess)
        return SDB_ERR_CUDA;
      ctc_marg_kernel<9><<<g, kMargWarps * 32, msmem, s>>>(ws.wsa, ws.wsabase, ws.wsb, ws.wsbase, logz, ws.csr, T, V,
                                                          L, status, marg);
    } else {
      if (msmem > 48 * 1024 && sdb_set_smem((const void*)ctc_marg_kernel<32>, msmem) != cudaSuccess)
        return SDB_ERR_CUDA;
      ctc_marg_kernel<32><<<g, kMargWarps * 32, msmem, s>>>(ws.wsa, ws.wsabase, ws.wsb, ws.wsbase, logz, ws.csr, T,
                                                           V, L, status, marg);
    }
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
