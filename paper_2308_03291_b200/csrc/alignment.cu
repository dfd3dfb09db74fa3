// Monotone (Needleman-Wunsch) alignment CRF: log-partition, move marginals,
// max-plus argmax.
//
// Reference: structdist alignment.py:62-143 (_nw_forward, _nw_backward,
// nw_marginals, _nw_walk, _nw_max_forward).  Moves are scored on arrival:
// DIAG=0 from (i-1,j-1), DOWN=1 from (i-1,j), RIGHT=2 from (i,j-1).
// Layout per instance: theta [n+1][m+1][3] fp32 row-major.
//
// Parallel schedule (one CTA per instance, NW = ceil((m+1)/32) warps):
//   * warp w owns a strip of 32 columns; lane l processes row i at local step
//     s = i + l (skewed wavefront), so its left neighbour (lane l-1) finished
//     the same row one step earlier -> warp shuffles, no barriers;
//   * warps are pipelined with a lag of LAG steps and exchange the strip
//     boundary column through a small shared ring; one __syncthreads every
//     kSync steps makes the ring visible (LAG = 32 + kSync - 1);
//   * potentials stream through a per-lane delay line in shared memory: at
//     step s every lane cp.async-loads row s+P of ITS column (the whole warp
//     loads one contiguous 384-byte row segment -> coalesced) and consumes
//     row s-l from the delay line.  The marginal of a cell overwrites its
//     potential in the delay line and is written back, again one coalesced
//     row segment per step, 32 steps later;
//   * marginals: phase A runs the backward recurrence on the flipped grid
//     (columns padded to 32*NW so flipping maps warps/lanes onto mirrored
//     warps/lanes) and stores beta as fp32 offsets from a per-(warp,step)
//     fp64 base in the same strip-diagonal layout the forward pass reads;
//     phase B runs the forward recurrence and emits every marginal as
//     exp(t_k - M) * exp(M + beta - Z), reusing the lse's own exponentials.
//   Log values are carried in fp64 (exact sums); exp/log run in fp32 MUFU on
//   small differences.
#include "common.cuh"

namespace {

constexpr int kR = 48;      // delay-line rows per warp (> 32 + kP)
constexpr int kP = 8;       // prefetch distance in steps
constexpr int kSync = 4;    // __syncthreads every kSync global steps
constexpr int kLag = 32 + kSync - 1;
constexpr int kRB = 32;     // strip-boundary ring (rows)
constexpr int kRP = 16;     // beta prefetch ring (steps)

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ double shfl_up_d(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }

struct NwShared {
  float* ring;    // [NW][kR][3][32]
  double* bnd0;   // [NW][kRB]
  double* bnd1;   // [NW][kRB]
  float* bq;      // [NW][kRP][32]
  double* bqb;    // [NW][kRP]
};

__device__ NwShared nw_carve(char* base, int NW) {
  NwShared s;
  s.ring = (float*)base;
  base += (size_t)NW * kR * 96 * sizeof(float);
  s.bnd0 = (double*)base;
  base += (size_t)NW * kRB * sizeof(double);
  s.bnd1 = (double*)base;
  base += (size_t)NW * kRB * sizeof(double);
  s.bqb = (double*)base;
  base += (size_t)NW * kRP * sizeof(double);
  s.bq = (float*)base;
  return s;
}

size_t nw_smem_bytes(int NW) {
  return (size_t)NW * kR * 96 * 4 + (size_t)NW * kRB * 16 + (size_t)NW * kRP * 8 + (size_t)NW * kRP * 32 * 4;
}

// lse of three fp64 log terms; returns (M, e0, e1, e2, sum) with e_k = exp(t_k - M)
struct Lse3 {
  double M;
  float e0, e1, e2, s;
};
__device__ __forceinline__ Lse3 lse3(double t0, double t1, double t2) {
  Lse3 r;
  r.M = fmax(fmax(t0, t1), t2);
  if (r.M == ninfd()) {
    r.e0 = r.e1 = r.e2 = 0.f;
    r.s = 0.f;
  } else {
    r.e0 = ex2((float)(t0 - r.M) * SDB_LOG2E);
    r.e1 = ex2((float)(t1 - r.M) * SDB_LOG2E);
    r.e2 = ex2((float)(t2 - r.M) * SDB_LOG2E);
    r.s = r.e0 + r.e1 + r.e2;
  }
  return r;
}
__device__ __forceinline__ double lse3_val(const Lse3& r) {
  return r.M == ninfd() ? ninfd() : r.M + (double)(lg2(r.s) * SDB_LN2);
}

// ------------------------------------------------------------------------
// Phase A: backward recurrence on the flipped grid, push form.  Stores
// beta(i,j) as fp32 offsets in the forward strip-diagonal layout
// wsb[w][s][l] (+ fp64 base wsbase[w][s]); returns Z = beta(0,0) via *zsh.
// ------------------------------------------------------------------------
__device__ void nw_phase_backward(const float* __restrict__ th, int n, int m, int NW, NwShared sh,
                                  float* __restrict__ wsb, double* __restrict__ wsbase, double* zsh) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int mp = 32 * NW - 1;
  const int jf = 32 * w + l;      // flipped column
  const int jo = mp - jf;         // original column
  const bool col_ok = jo <= m;
  const int steps = n + 32;
  const int G = steps + (NW - 1) * kLag;
  const size_t rowstride = (size_t)(m + 1) * 3;
  float* ring = sh.ring + (size_t)w * kR * 96;
  const int wf = NW - 1 - w, lf = 31 - l;

  double pDn = ninfd(), pR = ninfd(), pD = ninfd(), savedD = ninfd();
  for (int g = -kP; g < G; ++g) {
    const int s = g - w * kLag;
    // prefetch flipped row s+kP (original row n-(s+kP)) of this lane's column
    {
      const int rp = s + kP;
      if (rp >= 0 && rp <= n && col_ok) {
        const float* src = th + (size_t)(n - rp) * rowstride + (size_t)jo * 3;
        float* dst = ring + (rp % kR) * 96 + l;
        cp_async4(dst, src);
        cp_async4(dst + 32, src + 1);
        cp_async4(dst + 64, src + 2);
      }
      cp_commit();
    }
    if (s >= 0 && s < steps) {
      cp_wait<kP>();
      const int ip = s - l;  // flipped row
      double recvR = shfl_up_d(pR), recvD = shfl_up_d(pD);
      if (l == 0) {
        if (w == 0 || ip < 0 || ip > n) {
          recvR = ninfd();
          recvD = ninfd();
        } else {
          recvR = sh.bnd0[w * kRB + (ip % kRB)];
          recvD = sh.bnd1[w * kRB + (ip % kRB)];
        }
      }
      const double inR = recvR, inD = savedD, inDn = pDn;
      savedD = recvD;
      double b = ninfd();
      const bool valid = ip >= 0 && ip <= n && col_ok;
      if (valid) {
        const int io = n - ip;
        const float* slot = ring + (ip % kR) * 96 + l;
        const float t0 = slot[0], t1 = slot[32], t2 = slot[64];
        if (io == n && jo == m) {
          b = 0.0;
        } else {
          Lse3 r = lse3(inD, inDn, inR);
          b = lse3_val(r);
        }
        pD = b + (double)t0;
        pDn = b + (double)t1;
        pR = b + (double)t2;
        if (io == 0 && jo == 0) *zsh = b;
      } else {
        pD = pDn = pR = ninfd();
      }
      if (l == 31 && w + 1 < NW && ip >= 0 && ip <= n) {
        sh.bnd0[(w + 1) * kRB + (ip % kRB)] = pR;
        sh.bnd1[(w + 1) * kRB + (ip % kRB)] = pD;
      }
      // store beta into the forward strip layout: fwd warp wf, step n+31-s, lane 31-l
      double base = warp_maxd(b);
      if (base == ninfd()) base = 0.0;
      const size_t sf = (size_t)(n + 31 - s);
      wsb[((size_t)wf * steps + sf) * 32 + lf] = (b == ninfd()) ? ninf() : (float)(b - base);
      if (l == 0) wsbase[(size_t)wf * steps + sf] = base;
    }
    if (((g + 1) % kSync) == 0) __syncthreads();
  }
  cp_wait<0>();
  __syncthreads();
}

// ------------------------------------------------------------------------
// Phase B: forward recurrence (pull form).  kMarg: emit marginals using the
// stored beta and Z.  kMax: max-plus with argmax choices (no marginals).
// ------------------------------------------------------------------------
template <bool kMarg, bool kMax>
__device__ void nw_phase_forward(const float* __restrict__ th, int n, int m, int NW, NwShared sh,
                                 const float* __restrict__ wsb, const double* __restrict__ wsbase, double Z,
                                 float* __restrict__ marg, int8_t* __restrict__ choice, double* out_last,
                                 int* bad_flag) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int j = 32 * w + l;
  const bool col_ok = j <= m;
  const int steps = n + 32;
  const int G = steps + 1 + (NW - 1) * kLag;
  const size_t rowstride = (size_t)(m + 1) * 3;
  float* ring = sh.ring + (size_t)w * kR * 96;
  float* bq = sh.bq + (size_t)w * kRP * 32;
  double* bqb = sh.bqb + (size_t)w * kRP;
  const bool zok = !(Z == ninfd());
  int bad = 0;

  double aprev = ninfd(), cur = ninfd(), lprev = ninfd();
  for (int g = -kP; g < G; ++g) {
    const int s = g - w * kLag;
    {
      const int rp = s + kP;
      if (rp >= 0 && rp <= n && col_ok) {
        const float* src = th + (size_t)rp * rowstride + (size_t)j * 3;
        float* dst = ring + (rp % kR) * 96 + l;
        cp_async4(dst, src);
        cp_async4(dst + 32, src + 1);
        cp_async4(dst + 64, src + 2);
      }
      if (kMarg && rp >= 0 && rp < steps) {
        cp_async4(bq + (rp % kRP) * 32 + l, wsb + ((size_t)w * steps + rp) * 32 + l);
        if (l == 0) cp_async8(bqb + (rp % kRP), wsbase + (size_t)w * steps + rp);
      }
      cp_commit();
    }
    if (s >= 0 && s <= steps) {
      cp_wait<kP>();
      if (s < steps) {
        const int i = s - l;
        double left = shfl_up_d(cur);
        if (l == 0) {
          left = (w == 0 || i < 0 || i > n) ? ninfd() : sh.bnd0[w * kRB + (i % kRB)];
        }
        const double diag = lprev;
        lprev = left;
        const bool valid = i >= 0 && i <= n && col_ok;
        double a = ninfd();
        if (valid) {
          float* slot = ring + (i % kR) * 96 + l;
          const float t0 = slot[0], t1 = slot[32], t2 = slot[64];
          bad |= bad_input(t0) | bad_input(t1) | bad_input(t2);
          const double c0 = diag + (double)t0, c1 = aprev + (double)t1, c2 = left + (double)t2;
          if (kMax) {
            int k = 0;
            double best = ninfd();
            // first maximum among in-grid sources in DIAG, DOWN, RIGHT order (alignment.py:121-136)
            bool first = true;
            if (i > 0 && j > 0) { best = c0; k = 0; first = false; }
            if (i > 0 && (first || c1 > best)) { best = c1; k = 1; first = false; }
            if (j > 0 && (first || c2 > best)) { best = c2; k = 2; first = false; }
            a = (i == 0 && j == 0) ? 0.0 : best;
            choice[((size_t)w * steps + s) * 32 + l] = (int8_t)k;
          } else if (i == 0 && j == 0) {
            a = 0.0;
            if (kMarg) slot[0] = slot[32] = slot[64] = 0.f;
          } else {
            Lse3 r = lse3(c0, c1, c2);
            a = lse3_val(r);
            if (kMarg) {
              const float bt = bq[(s % kRP) * 32 + l];
              const double bb = bqb[s % kRP];
              float F = 0.f;
              if (zok && r.M != ninfd() && bt != ninf()) F = ex2(((float)(r.M + bb - Z) + bt) * SDB_LOG2E);
              slot[0] = r.e0 * F;
              slot[32] = r.e1 * F;
              slot[64] = r.e2 * F;
            }
          }
          aprev = a;
          if (i == n && j == m) *out_last = a;
        }
        cur = valid ? a : ninfd();
        if (l == 31 && w + 1 < NW && i >= 0 && i <= n) sh.bnd0[(w + 1) * kRB + (i % kRB)] = cur;
      }
      if (kMarg) {
        const int r = s - 32;  // row completed by every lane of this warp
        if (r >= 0 && r <= n && col_ok) {
          const float* slot = ring + (r % kR) * 96 + l;
          float* dst = marg + (size_t)r * rowstride + (size_t)j * 3;
          dst[0] = slot[0];
          dst[1] = slot[32];
          dst[2] = slot[64];
        }
      }
    }
    if (((g + 1) % kSync) == 0) __syncthreads();
  }
  cp_wait<0>();
  if (bad) atomicOr(bad_flag, 1);
}

// grid B, block 32*NW
template <int kMode>  // 0 = logZ only, 1 = logZ + marginals, 2 = max-plus argmax
__global__ void nw_kernel(const float* __restrict__ theta, int n, int m, float* __restrict__ wsb_all,
                          double* __restrict__ wsbase_all, int8_t* __restrict__ choice_all,
                          double* __restrict__ logz, float* __restrict__ marg_all, int32_t* __restrict__ path,
                          double* __restrict__ score, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) char smraw[];
  __shared__ double zsh, lastsh;
  __shared__ int badsh;
  const int NW = blockDim.x >> 5;
  const int b = blockIdx.x;
  NwShared sh = nw_carve(smraw, NW);
  const float* th = theta + (size_t)b * (n + 1) * (m + 1) * 3;
  const int steps = n + 32;
  const size_t wsz = (size_t)NW * steps;
  if (threadIdx.x == 0) {
    zsh = ninfd();
    lastsh = ninfd();
    badsh = 0;
  }
  __syncthreads();
  if (kMode == 1) {
    float* wsb = wsb_all + (size_t)b * wsz * 32;
    double* wsbase = wsbase_all + (size_t)b * wsz;
    nw_phase_backward(th, n, m, NW, sh, wsb, wsbase, &zsh);
    __syncthreads();
    nw_phase_forward<true, false>(th, n, m, NW, sh, wsb, wsbase, zsh,
                                  marg_all + (size_t)b * (n + 1) * (m + 1) * 3, nullptr, &lastsh, &badsh);
  } else if (kMode == 0) {
    nw_phase_forward<false, false>(th, n, m, NW, sh, nullptr, nullptr, 0.0, nullptr, nullptr, &lastsh, &badsh);
  } else {
    int8_t* ch = choice_all + (size_t)b * wsz * 32;
    nw_phase_forward<false, true>(th, n, m, NW, sh, nullptr, nullptr, 0.0, nullptr, ch, &lastsh, &badsh);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double z = lastsh;
    const int st = badsh ? SDB_ST_INVALID : (z == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
    status[b] = st;
    if (kMode == 2) {
      score[b] = z;
    } else {
      logz[b] = z;
    }
  }
}

// backtrack kernel for the max-plus path: one thread per instance walks the
// choices (strip layout) from (n, m) to (0, 0) and marks the path.
__global__ void nw_walk_kernel(const int8_t* __restrict__ choice_all, int n, int m, int NW, int64_t B,
                               const int32_t* __restrict__ status, int8_t* __restrict__ path_all) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (status[b] != SDB_ST_OK) return;
  const int steps = n + 32;
  const int8_t* ch = choice_all + (size_t)b * NW * steps * 32;
  int8_t* pb = path_all + (size_t)b * (n + 1) * (m + 1);
  int i = n, j = m;
  while (i != 0 || j != 0) {
    const int w = j >> 5, l = j & 31, s = i + l;
    const int k = ch[((size_t)w * steps + s) * 32 + l];
    pb[(size_t)i * (m + 1) + j] = (int8_t)k;
    if (k == 0) { --i; --j; } else if (k == 1) { --i; } else { --j; }
  }
}

struct NwWs {
  float* wsb;
  double* wsbase;
  int8_t* choice;
};

NwWs nw_carve_ws(void* base, int64_t B, int n, int m, int mode, size_t* bytes) {
  const int NW = (m + 1 + 31) / 32;
  const size_t wsz = (size_t)NW * (n + 32);
  Carve c(base);
  NwWs w{};
  if (mode == 1) {
    w.wsb = c.take<float>((size_t)B * wsz * 32);
    w.wsbase = c.take<double>((size_t)B * wsz);
  }
  if (mode == 2) w.choice = c.take<int8_t>((size_t)B * wsz * 32);
  *bytes = c.used;
  return w;
}

template <int kMode>
int nw_launch(const float* theta, int64_t B, int n, int m, NwWs ws, double* logz, float* marg, int8_t* path,
              double* score, int32_t* status, cudaStream_t s) {
  const int NW = (m + 1 + 31) / 32;
  const size_t smem = nw_smem_bytes(NW);
  if (cudaFuncSetAttribute(nw_kernel<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SDB_ERR_CUDA;
  nw_kernel<kMode><<<(unsigned)B, 32 * NW, smem, s>>>(theta, n, m, ws.wsb, ws.wsbase, ws.choice, logz, marg,
                                                      nullptr, score, status);
  SDB_CHECK_LAUNCH();
  if (kMode == 2) {
    nw_walk_kernel<<<(unsigned)((B + 127) / 128), 128, 0, s>>>(ws.choice, n, m, NW, B, status, path);
    SDB_CHECK_LAUNCH();
  }
  return SDB_OK;
}

int nw_check(int64_t B, int n, int m) {
  if (B < 0 || n < 1 || m < 1) return SDB_ERR_ARG;
  const int NW = (m + 1 + 31) / 32;
  if (NW > 32 || nw_smem_bytes(NW) > 220 * 1024) return SDB_ERR_UNSUPPORTED;
  return SDB_OK;
}

}  // namespace

extern "C" size_t sdb_nw_fb_workspace(int64_t B, int32_t n, int32_t m) {
  size_t bytes = 0;
  nw_carve_ws(nullptr, B, n, m, 1, &bytes);
  return bytes;
}

extern "C" int sdb_nw_fb(const float* theta, int64_t B, int32_t n, int32_t m, double* logz, float* marg,
                         int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  int rc = nw_check(B, n, m);
  if (rc) return rc;
  if (!theta || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!marg) return nw_launch<0>(theta, B, n, m, NwWs{}, logz, nullptr, nullptr, nullptr, status, (cudaStream_t)stream);
  size_t need = 0;
  NwWs ws = nw_carve_ws(workspace, B, n, m, 1, &need);
  if (!workspace || ws_bytes < need) return SDB_ERR_WORKSPACE;
  return nw_launch<1>(theta, B, n, m, ws, logz, marg, nullptr, nullptr, status, (cudaStream_t)stream);
}

extern "C" size_t sdb_nw_viterbi_workspace(int64_t B, int32_t n, int32_t m) {
  size_t bytes = 0;
  nw_carve_ws(nullptr, B, n, m, 2, &bytes);
  return bytes;
}

extern "C" int sdb_nw_viterbi(const float* theta, int64_t B, int32_t n, int32_t m, int8_t* path, double* score,
                              int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  int rc = nw_check(B, n, m);
  if (rc) return rc;
  if (!theta || !path || !score || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  size_t need = 0;
  NwWs ws = nw_carve_ws(workspace, B, n, m, 2, &need);
  if (!workspace || ws_bytes < need) return SDB_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(path, 0xff, (size_t)B * (n + 1) * (m + 1), s) != cudaSuccess) return SDB_ERR_CUDA;
  return nw_launch<2>(theta, B, n, m, ws, nullptr, nullptr, path, score, status, s);
}
