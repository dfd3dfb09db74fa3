// CTC over the blank-interleaved 2L+1 lattice: log-partition, per-frame
// vocabulary marginals, best expanded-state path.
//
// Reference: structdist alignment.py:231-336 (_expanded_labels,
// _ctc_predecessors, _ctc_forward, _ctc_backward, ctc_marginals, ctc_argmax,
// _ctc_walk).  Layout per instance: frame_potentials [T][V] fp32,
// targets [L] int32 (labels in 1..V-1), blank = 0.
//
// Schedule: one CTA per instance, one thread per lattice state s (S = 2L+1
// <= 1024), frames in lockstep (one __syncthreads per frame).  Frame rows are
// prefetched kP frames ahead into a shared ring with cp.async and each state
// gathers its emission theta[t][lab(s)] from shared memory.
//   phase A: beta over frames T-1..0, stored as fp32 offsets from a per-frame
//            fp64 base (the frame max) -> workspace; Z = lse(beta[0][0..1] + E).
//   phase B: alpha over frames 0..T-1; posterior exp(alpha + beta - Z) per
//            state, reduced by label deterministically (blank: fixed-order warp
//            butterflies; labels: each vocabulary thread sums its own state
//            list in increasing s) and written as one coalesced [V] row.
// Log values are fp64; exp/log fp32 MUFU on differences.
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
  double* a0;     // [S+2] ping (2 leading -inf pads)
  double* a1;     // [S+2] pong
  float* rows;    // [kP][V]
  int* lab;       // [S]
  int* lst;       // [L] states grouped by label (CSR)
  int* off;       // [V+1]
  float* post;    // [S]
  double* wred;   // [2][32]
  float* bred;    // [32]
  float* bring;   // [kP][S] beta rows (phase B prefetch)
  double* bbase;  // [kP][32] their per-warp bases
};

size_t ctc_smem_bytes(int S, int V, int L) {
  return (size_t)2 * (S + 2) * 8 + (size_t)kP * V * 4 + (size_t)S * 4 + (size_t)(L + 1) * 4 +
         (size_t)(V + 1) * 4 + (size_t)S * 4 + 64 * 8 + 32 * 4 + (size_t)kP * 32 * 8 + (size_t)kP * S * 4 + 128;
}

__device__ CtcSmem ctc_carve(char* p, int S, int V, int L) {
  CtcSmem s;
  s.a0 = (double*)p; p += (size_t)(S + 2) * 8;
  s.a1 = (double*)p; p += (size_t)(S + 2) * 8;
  s.wred = (double*)p; p += 64 * 8;
  s.bbase = (double*)p; p += kP * 32 * 8;
  s.rows = (float*)p; p += (size_t)kP * V * 4;
  s.lab = (int*)p; p += (size_t)S * 4;
  s.lst = (int*)p; p += (size_t)(L + 1) * 4;
  s.off = (int*)p; p += (size_t)(V + 1) * 4;
  s.post = (float*)p; p += (size_t)S * 4;
  s.bred = (float*)p; p += 32 * 4;
  s.bring = (float*)p;
  return s;
}

__device__ __forceinline__ void load_row(const float* __restrict__ fp, int t, int V, float* dst) {
  for (int v = threadIdx.x; v < V; v += blockDim.x) cp_async4(dst + v, fp + (size_t)t * V + v);
}

template <int kMode>  // 0 logZ only, 1 logZ + marginals, 2 max-plus path
__global__ void ctc_kernel(const float* __restrict__ fp_all, const int32_t* __restrict__ tg_all, int T, int V,
                           int L, float* __restrict__ wsb_all, double* __restrict__ wsbase_all,
                           int32_t* __restrict__ csr_all, int8_t* __restrict__ back_all, double* __restrict__ logz, float* __restrict__ marg_all,
                           int32_t* __restrict__ path_all, double* __restrict__ score,
                           int32_t* __restrict__ status) {
  extern __shared__ __align__(16) char smraw[];
  const int S = 2 * L + 1;
  CtcSmem sm = ctc_carve(smraw, S, V, L);
  __shared__ double zsh;
  __shared__ int badsh;
  const int b = blockIdx.x, tid = threadIdx.x;
  const float* fp = fp_all + (size_t)b * T * V;
  const int32_t* tg = tg_all + (size_t)b * L;
  const int s = tid;
  const bool act = s < S;

  // ---- prologue: labels, skip flags, label lists
  if (tid == 0) {
    badsh = 0;
    zsh = ninfd();
  }
  __syncthreads();
  int mylab = 0;
  bool skip = false;
  if (act) {
    mylab = (s & 1) ? tg[s >> 1] : 0;
    if ((s & 1) && (mylab < 1 || mylab >= V)) {
      atomicOr(&badsh, 1);
      mylab = 0;
    }
    sm.lab[s] = mylab;
  }
  __syncthreads();
  if (act) skip = (s >= 2) && mylab != 0 && mylab != sm.lab[s - 2];
  if (kMode == 1) {
    if (tid == 0) {  // CSR of the odd states by label, increasing s (deterministic order)
      for (int v = 0; v <= V; ++v) sm.off[v] = 0;
      for (int k = 0; k < L; ++k) sm.off[sm.lab[2 * k + 1] + 1]++;
      for (int v = 0; v < V; ++v) sm.off[v + 1] += sm.off[v];
      for (int k = 0; k < L; ++k) sm.lst[k] = -1;
      for (int k = 0; k < L; ++k) {
        int pos = sm.off[sm.lab[2 * k + 1]];
        while (sm.lst[pos] >= 0) ++pos;
        sm.lst[pos] = 2 * k + 1;
      }
    }
    __syncthreads();
  }
  const int nwarps = blockDim.x >> 5;
  (void)nwarps;
  float* wsb = (kMode == 1) ? wsb_all + (size_t)b * T * S : nullptr;
  if (kMode == 1) {  // the label CSR, for ctc_marg_kernel
    int32_t* csr = csr_all + (size_t)b * (V + 1 + L);
    for (int e = tid; e <= V; e += blockDim.x) csr[e] = sm.off[e];
    for (int e = tid; e < L; e += blockDim.x) csr[V + 1 + e] = sm.lst[e];
  }
  double* wsbase = (kMode == 1) ? wsbase_all + (size_t)b * T * 32 : nullptr;  // [T][32 warps]

  // ======================= phase A: backward (marginals only)
  if (kMode == 1) {
    double* cur = sm.a0 + 2;  // beta[t+1][*]
    double* nxt = sm.a1 + 2;
    // prefetch frames T-1 .. T-kP (we need E[t+1] while computing beta[t])
    for (int k = 0; k < kP; ++k) {
      const int t = T - 1 - k;
      if (t >= 0) load_row(fp, t, V, sm.rows + (size_t)(t % kP) * V);
      cp_commit();
    }
    if (act) cur[s] = (s == S - 1 || s == S - 2) ? 0.0 : ninfd();
    if (tid < S + 2 && tid >= S) cur[tid] = ninfd();  // right pads beyond S
    if (tid < 2) { sm.a0[tid] = ninfd(); sm.a1[tid] = ninfd(); }
    __syncthreads();
    // store beta[T-1] (offsets from a per-WARP base: a warp max, no CTA reduction per frame)
    {
      const double v = act ? cur[s] : ninfd();
      const float wm = warp_max((float)v);
      const double base = (wm == ninf()) ? 0.0 : (double)wm;
      if (act) wsb[(size_t)(T - 1) * S + s] = (v == ninfd()) ? ninf() : (float)(v - base);
      if ((tid & 31) == 0) wsbase[(size_t)(T - 1) * 32 + (tid >> 5)] = base;
    }
    // successor labels of this state are fixed for all frames: keep them in registers
    const bool has1 = act && (s + 1 < S);
    const int lab1 = has1 ? sm.lab[s + 1] : 0;
    const int lab2 = (act && s + 2 < S) ? sm.lab[s + 2] : 0;
    const bool sk2 = act && (s + 2 < S) && lab2 != 0 && lab2 != mylab;
    for (int t = T - 2; t >= 0; --t) {
      // frame t+1 must be resident: it was issued (T-1)-(t+1) groups ago
      cp_wait<kP - 1>();
      __syncthreads();
      const float* E = sm.rows + (size_t)((t + 1) % kP) * V;
      double v = ninfd();
      if (act) {
        const double x0 = cur[s] + (double)E[mylab];
        const double x1 = has1 ? cur[s + 1] + (double)E[lab1] : ninfd();
        const double x2 = sk2 ? cur[s + 2] + (double)E[lab2] : ninfd();
        const double M = fmax(fmax(x0, x1), x2);
        if (M != ninfd()) {
          const float e = fexp((float)(x0 - M)) + fexp((float)(x1 - M)) + fexp((float)(x2 - M));
          v = M + (double)flog(e);
        }
        nxt[s] = v;
      }
      // beta[t] as fp32 offsets from its warp's max (the base only has to be close to the
      // values it is subtracted from; one fp32 warp max, no CTA-wide reduction)
      {
        const float wm = warp_max((float)v);
        const double base = (wm == ninf()) ? 0.0 : (double)wm;
        if (act) wsb[(size_t)t * S + s] = (v == ninfd()) ? ninf() : (float)(v - base);
        if ((tid & 31) == 0) wsbase[(size_t)t * 32 + (tid >> 5)] = base;
      }
      __syncthreads();  // all reads of cur and row (t+1) done; nxt complete
      // refill the ring slot of frame t+1 with frame t+1-kP
      {
        const int tn = t + 1 - kP;
        if (tn >= 0) load_row(fp, tn, V, sm.rows + (size_t)(tn % kP) * V);
        cp_commit();
      }
      double* tmp = cur; cur = nxt; nxt = tmp;
    }
    cp_wait<0>();
    __syncthreads();
    // Z = lse(beta[0][0] + E0[lab0], beta[0][1] + E0[lab1])  (E0 = frame 0 still in the ring)
    if (tid == 0) {
      const float* E0 = sm.rows;  // frame 0 sits in slot 0
      const double z0 = cur[0] + (double)E0[sm.lab[0]];
      const double z1 = (S > 1) ? cur[1] + (double)E0[sm.lab[1]] : ninfd();
      const double M = fmax(z0, z1);
      zsh = (M == ninfd()) ? ninfd() : M + (double)flog(fexp((float)(z0 - M)) + fexp((float)(z1 - M)));
    }
    __syncthreads();
  }

  // ======================= phase B: forward
  {
    double* prv = sm.a0 + 2;  // alpha[t-1]
    double* now = sm.a1 + 2;
    if (tid < 2) { sm.a0[tid] = ninfd(); sm.a1[tid] = ninfd(); }
    auto load_beta = [&](int t) {  // beta row t + its base into ring slot t % kP
      if (kMode != 1) return;
      if (act) cp_async4(sm.bring + (size_t)(t % kP) * S + s, wsb + (size_t)t * S + s);
      if ((tid & 31) == 0) {  // this warp's base
        unsigned sa = (unsigned)__cvta_generic_to_shared(sm.bbase + (t % kP) * 32 + (tid >> 5));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(wsbase + (size_t)t * 32 + (tid >> 5)));
      }
    };
    for (int k = 0; k < kP; ++k) {
      if (k < T) {
        load_row(fp, k, V, sm.rows + (size_t)k * V);
        load_beta(k);
      }
      cp_commit();
    }
    const double Z = zsh;
    const bool zok = Z != ninfd();
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
      if (kMode == 1 && act) {
        // posterior of state s at frame t, written over beta's slot (frame t of the beta ring
        // has been consumed); ctc_marg_kernel scatter-adds the rows by label off this loop
        float p = 0.f;
        if (zok && a != ninfd()) {
          const float bt = sm.bring[(size_t)(t % kP) * S + s];
          const double bb = sm.bbase[(t % kP) * 32 + (tid >> 5)];
          if (bt != ninf()) p = fexp((float)(a + bb - Z) + bt);
        }
        wsb[(size_t)t * S + s] = p;
      }
      __syncthreads();  // now[] complete; row t consumed
      {
        const int tn = t + kP;
        if (tn < T) {
          load_row(fp, tn, V, sm.rows + (size_t)(tn % kP) * V);
          load_beta(tn);
        }
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
}

// Per-frame vocabulary marginals from the posteriors ctc_kernel<1> left in
// the workspace (alignment.py:290-301): marg[t][v] = sum of post[t][s] over
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
__global__ void __launch_bounds__(kMargWarps * 32) ctc_marg_kernel(const float* __restrict__ post_all,
                                                                  const int32_t* __restrict__ csr_all, int T, int V,
                                                                  int L, const int32_t* __restrict__ status,
                                                                  float* __restrict__ marg_all) {
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
  const int32_t* csr = csr_all + (size_t)b * (V + 1 + L);  // built by ctc_kernel<1>
  for (int e = tid; e <= V; e += blockDim.x) off[e] = csr[e];
  for (int e = tid; e < L; e += blockDim.x) lst[e] = csr[V + 1 + e];
  __syncthreads();
  float* prow = prow_all + (size_t)warp * S;
  const float* pb = post_all + (size_t)b * T * S;
  // the warp's next frame is loaded into registers while the current one is reduced
  float nxt[kRowRegs];
  auto fetch = [&](int t) {
    const float* src = pb + (size_t)t * S;
#pragma unroll
    for (int u = 0; u < kRowRegs; ++u) {
      const int e = lane + 32 * u;
      if (e < S) nxt[u] = src[e];
    }
  };
  if (t0 + warp < t1) fetch(t0 + warp);
  for (int t = t0 + warp; t < t1; t += kMargWarps) {
#pragma unroll
    for (int u = 0; u < kRowRegs; ++u) {
      const int e = lane + 32 * u;
      if (e < S) prow[e] = nxt[u];
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
  float* wsb;      // [B][T][S] beta offsets, then the state posteriors
  double* wsbase;  // [B][T][32] per-warp beta bases
  int32_t* csr;    // [B][V+1+L] label CSR (offsets, odd states by label)
  int8_t* back;
};

CtcWs ctc_carve_ws(void* base, int64_t B, int T, int V, int L, int mode, size_t* bytes) {
  const int S = 2 * L + 1;
  Carve c(base);
  CtcWs w{};
  if (mode == 1) {
    w.wsb = c.take<float>((size_t)B * T * S);
    w.wsbase = c.take<double>((size_t)B * T * 32);
    w.csr = c.take<int32_t>((size_t)B * (V + 1 + L));
  }
  if (mode == 2) w.back = c.take<int8_t>((size_t)B * T * S);
  *bytes = c.used;
  return w;
}

int ctc_check(int64_t B, int T, int V, int L) {
  if (B < 0 || T < 1 || V < 1 || L < 0) return SDB_ERR_ARG;
  const int S = 2 * L + 1;
  if (S > 1024 || ctc_smem_bytes(S, V, L) > 200 * 1024) return SDB_ERR_UNSUPPORTED;
  return SDB_OK;
}

template <int kMode>
int ctc_launch(const float* fp, const int32_t* tg, int64_t B, int T, int V, int L, CtcWs ws, double* logz,
               float* marg, int32_t* path, double* score, int32_t* status, cudaStream_t s) {
  const int S = 2 * L + 1;
  const int threads = ((S + 31) / 32) * 32;
  const size_t smem = ctc_smem_bytes(S, V, L);
  if (cudaFuncSetAttribute(ctc_kernel<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SDB_ERR_CUDA;
  ctc_kernel<kMode><<<(unsigned)B, threads, smem, s>>>(fp, tg, T, V, L, ws.wsb, ws.wsbase, ws.csr, ws.back, logz,
                                                      marg, path, score, status);
  SDB_CHECK_LAUNCH();
  if (kMode == 1) {
    const int S2 = 2 * L + 1;
    const size_t msmem = (((size_t)(V + 1 + L) + 3) & ~(size_t)3) * 4 + (size_t)kMargWarps * S2 * 4;
    dim3 g((unsigned)((T + kMargFrames - 1) / kMargFrames), (unsigned)B);
    const int rr = (S2 + 31) / 32;
    if (rr <= 9) {
      if (msmem > 48 * 1024 && cudaFuncSetAttribute(ctc_marg_kernel<9>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    (int)msmem) != cudaSuccess)
        return SDB_ERR_CUDA;
      ctc_marg_kernel<9><<<g, kMargWarps * 32, msmem, s>>>(ws.wsb, ws.csr, T, V, L, status, marg);
    } else {
      if (msmem > 48 * 1024 && cudaFuncSetAttribute(ctc_marg_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    (int)msmem) != cudaSuccess)
        return SDB_ERR_CUDA;
      ctc_marg_kernel<32><<<g, kMargWarps * 32, msmem, s>>>(ws.wsb, ws.csr, T, V, L, status, marg);
    }
    SDB_CHECK_LAUNCH();
  }
  return SDB_OK;
}

}  // namespace

extern "C" size_t sdb_ctc_fb_workspace(int64_t B, int32_t T, int32_t V, int32_t L) {
  (void)V;
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
  if (!marg) return ctc_launch<0>(frame_potentials, targets, B, T, V, L, CtcWs{}, logz, nullptr, nullptr, nullptr, status, s);
  size_t need = 0;
  CtcWs ws = ctc_carve_ws(workspace, B, T, V, L, 1, &need);
  if (!workspace || ws_bytes < need) return SDB_ERR_WORKSPACE;
  return ctc_launch<1>(frame_potentials, targets, B, T, V, L, ws, logz, marg, nullptr, nullptr, status, s);
}

extern "C" size_t sdb_ctc_viterbi_workspace(int64_t B, int32_t T, int32_t V, int32_t L) {
  (void)V;
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
  size_t need = 0;
  CtcWs ws = ctc_carve_ws(workspace, B, T, V, L, 2, &need);
  if (!workspace || ws_bytes < need) return SDB_ERR_WORKSPACE;
  return ctc_launch<2>(frame_potentials, targets, B, T, V, L, ws, nullptr, nullptr, labels, score, status,
                       (cudaStream_t)stream);
}
