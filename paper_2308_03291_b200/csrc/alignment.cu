// Monotone (Needleman-Wunsch) alignment CRF: log-partition, move marginals,
// max-plus argmax.
//
// Reference: structdist alignment.py:62-167 (_nw_forward, _nw_backward,
// nw_marginals, _nw_walk, _nw_max_forward, nw_argmax).  Moves are scored on
// arrival: DIAG=0 from (i-1,j-1), DOWN=1 from (i-1,j), RIGHT=2 from (i,j-1).
// Layout per instance: theta [n+1][m+1][3] fp32 row-major.
//
// Schedule (one CTA per instance, NW = ceil((m+1)/32) warps):
//   * warp w owns a strip of 32 columns; lane l processes row i at local step
//     s = i + l (skewed wavefront), so its left neighbour (lane l-1) finished
//     the same row one step earlier -> one warp shuffle per step, no barrier;
//   * warps are pipelined with a lag of kLag steps and exchange the strip
//     boundary column through a small shared ring; one __syncthreads per
//     8-step block makes it visible (lag >= 32 + 7).  (A flag-based
//     producer/consumer variant without barriers measured 3x slower: the
//     CTA fence waits on the in-flight cp.async prefetches.);
//   * potentials stream through a per-lane delay line in shared memory: at
//     step s every lane cp.async-loads row s+8 of ITS column (the whole warp
//     loads one contiguous 384-byte row segment -> coalesced) and consumes
//     row s-l.  A cell's marginals overwrite its potentials in the delay line
//     and are written back 32 steps later, again as one row segment;
//   * log values are fp32 in log2 units carried as (v, O), value = v + O with
//     an integer offset O re-chosen every step (O += rint(max)); messages carry
//     their offset and receivers convert with an exact integer difference, so
//     no fp64 and no precision loss at |log Z| ~ 10^3;
//   * marginals: phase A runs the backward recurrence on the flipped grid
//     (columns padded to 32*NW so flipping maps warps/lanes onto mirrored
//     warps/lanes) and stores beta as fp32 offsets from a per-(warp,step)
//     integer reference in the strip layout the forward pass reads; phase B
//     runs the forward recurrence and emits e_k * exp2(M + beta - Z) from the
//     lse's own exponentials.
// The max-plus argmax runs the same skew in fp64 (exact sums in the
// reference's order) with per-cell argmax choices and a backtrack kernel.
#include "common.cuh"

namespace {

constexpr int kR = 48;    // delay-line rows per warp (> 32 + kP, multiple of kBlk)
constexpr int kP = 8;     // prefetch distance in steps
constexpr int kBlk = 8;   // steps per progress-publication block
constexpr int kRB = 64;   // strip-boundary ring rows
constexpr int kRP = 16;   // beta prefetch ring (steps)
constexpr int kLag = 40;  // warp-to-warp lag: >= 32 + kBlk - 1 and a multiple of kBlk, so every warp
                          // reaches the per-block barrier at the same phase of its own schedule
static_assert(kR % kBlk == 0 && kP % kBlk == 0 && kLag % kBlk == 0 && kLag >= 32 + kBlk - 1, "alignment");

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp4p(uint32_t saddr, const void* gmem, bool pred) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p cp.async.ca.shared.global [%0], [%1], 4;\n}\n" ::"r"(saddr),
      "l"(gmem), "r"((int)pred));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__device__ __forceinline__ int mod_pos(int x, int R) {
  const int r = x % R;
  return r < 0 ? r + R : r;
}

struct NwShared {
  float* ring;   // [NW][kR][3][32]
  float2* bnd0;  // [NW][kRB]
  float2* bnd1;  // [NW][kRB]
  float* bq;     // [NW][kRP][32]
  float* bk;     // [NW][kRP]
  int* prog;     // [NW] last completed local step
};

__device__ NwShared nw_carve(char* base, int NW) {
  NwShared s;
  s.ring = (float*)base;
  base += (size_t)NW * kR * 96 * 4;
  s.bnd0 = (float2*)base;
  base += (size_t)NW * kRB * 8;
  s.bnd1 = (float2*)base;
  base += (size_t)NW * kRB * 8;
  s.bq = (float*)base;
  base += (size_t)NW * kRP * 32 * 4;
  s.bk = (float*)base;
  base += (size_t)NW * kRP * 4;
  s.prog = (int*)base;
  return s;
}

size_t nw_smem_bytes(int NW) {
  return (size_t)NW * kR * 96 * 4 + (size_t)NW * kRB * 16 + (size_t)NW * kRP * 33 * 4 + (size_t)NW * 4 + 64;
}

struct VO {
  float v, o;
};
__device__ __forceinline__ float rel(VO x, float o) { return x.v + (x.o - o); }

// log-sum-exp of three log2-unit terms, branch-free: value in the frame
// shifted by r = rint(M) (exact); e_k = exp2(t_k - Mc).  All -inf -> -inf, r = 0.
struct L3 {
  float v, r, Mc, e0, e1, e2;
};
__device__ __forceinline__ L3 lse3r(float t0, float t1, float t2) {
  L3 o;
  const float M = fmaxf(fmaxf(t0, t1), t2);
  o.Mc = fmaxf(M, -1e30f);
  o.r = (M > -1e30f) ? rintf(M) : 0.f;
  o.e0 = ex2(t0 - o.Mc);
  o.e1 = ex2(t1 - o.Mc);
  o.e2 = ex2(t2 - o.Mc);
  o.v = (o.Mc - o.r) + lg2(o.e0 + o.e1 + o.e2);  // lg2(0) = -inf
  return o;
}

template <bool B>
struct BoolC {
  static constexpr bool value = B;
};

// A block of kBlk steps is "steady" when every lane's cell is strictly
// inside the grid rows (1 <= i < n), every prefetch row exists and no step
// touches the start/end cell: the step then needs no row/origin predicates.
// Steady blocks are the bulk of the work for n >> 32 and run a branch-free
// straight-line body the compiler can interleave across the 8 steps.
__device__ __forceinline__ bool steady_block(int s0, int n) { return (s0 >= 32) & (s0 + kBlk - 1 + kP < n); }

// =========================================================== phase A
// Backward recurrence on the flipped grid (push form).  Stores beta(i,j) as
// wsb[w][s][l] = b + (O - K[w][s]) in the FORWARD strip layout (K = a per
// (warp, step) integer reference: the warp max of the lane offsets on edge
// blocks, lane 31's offset on steady blocks -- lane 31 always owns a real
// column); returns Z = beta(0,0) as (zint, zfrac).
template <bool kCheck>
__device__ void nw_backward(const float* __restrict__ th, int n, int m, int NW, const NwShared& sh,
                            float* __restrict__ wsb, float* __restrict__ wsk, float* zint, float* zfrac,
                            int* bad_flag) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int mp = 32 * NW - 1;
  const int jo = mp - (32 * w + l);
  const bool col_ok = jo <= m;
  const int steps = n + 32;
  const int nblk = (steps + (NW - 1) * kLag + kP + kBlk - 1) / kBlk;
  const size_t rowstride = (size_t)(m + 1) * 3;
  const uint32_t ring_u = smem_u32(sh.ring + (size_t)w * kR * 96) + 4u * l;
  const float* ring_l = sh.ring + (size_t)w * kR * 96 + l;
  const int wf = NW - 1 - w, lf = 31 - l;
  const float* src_col = th + (size_t)(col_ok ? jo : m) * 3;
  const float2* bnd0_in = sh.bnd0 + w * kRB;
  const float2* bnd1_in = sh.bnd1 + w * kRB;
  float2* bnd0_out = sh.bnd0 + (w + 1) * kRB;
  float2* bnd1_out = sh.bnd1 + (w + 1) * kRB;
  const bool pub = (l == 31) & (w + 1 < NW);
  VO pDn{ninf(), 0.f}, pR{ninf(), 0.f}, pD{ninf(), 0.f}, savedD{ninf(), 0.f};
  float O = 0.f;
  bool bad = false;
  for (int blk = 0; blk < nblk; ++blk) {
    const int s0 = -kP - w * kLag + blk * kBlk;
    if ((s0 + kBlk - 1 < -kP) | (s0 >= steps)) {  // pipeline fill/drain: nothing to load or compute
      __syncthreads();
      continue;
    }
    const int pbase = mod_pos(s0 + kP, kR);
    const int cbase = mod_pos(s0 - l, kR);
    const int b0 = s0 & (kRB - 1);  // s0 is a multiple of kBlk: b0 + k never wraps
    float* wsb_blk = wsb + ((size_t)wf * steps + (size_t)(n + 31 - s0)) * 32 + lf;
    float* wsk_blk = wsk + (size_t)wf * steps + (size_t)(n + 31 - s0);
    auto step = [&](auto steady_c, int k) {
      constexpr bool kS = decltype(steady_c)::value;
      const int s = s0 + k;
      {  // prefetch flipped row s + kP (original row n - (s + kP)) of this lane's column
        const int rp = s + kP;
        const bool pv = kS ? true : ((rp >= 0) & (rp <= n));
        const float* src = src_col + (size_t)(pv ? n - rp : 0) * rowstride;
        const uint32_t dst = ring_u + (uint32_t)(pbase + k) * 384u;
        cp4p(dst, src, pv);
        cp4p(dst + 128, src + 1, pv);
        cp4p(dst + 256, src + 2, pv);
        cp_commit();
      }
      if (kS || (s >= 0 && s < steps)) {
        cp_wait<kP>();
        const int ip = s - l;
        VO rR, rD;
        rR.v = __shfl_up_sync(0xffffffffu, pR.v, 1);
        rR.o = __shfl_up_sync(0xffffffffu, pR.o, 1);
        rD.v = __shfl_up_sync(0xffffffffu, pD.v, 1);
        rD.o = __shfl_up_sync(0xffffffffu, pD.o, 1);
        const bool inrow = kS ? true : ((ip >= 0) & (ip <= n));
        {  // lane 0 pulls the neighbour strip's boundary (broadcast read by all lanes)
          const float2 a = bnd0_in[b0 + k], d = bnd1_in[b0 + k];
          const bool ok = (w > 0) & inrow;
          const bool l0 = l == 0;
          rR.v = l0 ? (ok ? a.x : ninf()) : rR.v;
          rR.o = l0 ? (ok ? a.y : 0.f) : rR.o;
          rD.v = l0 ? (ok ? d.x : ninf()) : rD.v;
          rD.o = l0 ? (ok ? d.y : 0.f) : rD.o;
        }
        const VO inR = rR, inD = savedD, inDn = pDn;
        savedD = rD;
        const bool valid = inrow & col_ok;
        int cs = cbase + k;
        cs -= (cs >= kR) ? kR : 0;
        const float* slot = ring_l + cs * 96;
        float x0 = slot[0], x1 = slot[32], x2 = slot[64];
        if (kCheck) bad |= valid & (bad_input(x0) | bad_input(x1) | bad_input(x2));
        if (!kS) {  // slots of cells outside the grid were never loaded: keep their pushes -inf, not NaN
          x0 = valid ? x0 : 0.f;
          x1 = valid ? x1 : 0.f;
          x2 = valid ? x2 : 0.f;
        }
        const L3 r = lse3r(rel(inD, O), rel(inDn, O), rel(inR, O));
        float b;
        if (kS) {
          b = r.v;
          O = O + r.r;
        } else {
          const bool start = (ip == 0) & (jo == m);  // original cell (n, m)
          b = start ? 0.f : r.v;
          O = start ? 0.f : O + r.r;
        }
        b = valid ? b : ninf();
        pD = VO{fmaf(x0, SDB_LOG2E, b), O};
        pDn = VO{fmaf(x1, SDB_LOG2E, b), O};
        pR = VO{fmaf(x2, SDB_LOG2E, b), O};
        if (!kS && valid && ip == n && jo == 0) {
          *zint = O;
          *zfrac = b;
        }
        if (pub & inrow) {
          bnd0_out[(ip & (kRB - 1))] = make_float2(pR.v, pR.o);
          bnd1_out[(ip & (kRB - 1))] = make_float2(pD.v, pD.o);
        }
        float K;
        if (kS) {
          K = __shfl_sync(0xffffffffu, O, 31);
        } else {
          const float K0 = warp_max(b == ninf() ? ninf() : O);
          K = (K0 == ninf()) ? 0.f : K0;
        }
        wsb_blk[-32 * k] = (b == ninf()) ? ninf() : b + (O - K);
        if (l == 0) wsk_blk[-k] = K;
      }
    };
    if (steady_block(s0, n)) {
#pragma unroll
      for (int k = 0; k < kBlk; ++k) step(BoolC<true>{}, k);
    } else {
#pragma unroll
      for (int k = 0; k < kBlk; ++k) step(BoolC<false>{}, k);
    }
    __syncthreads();
  }
  cp_wait<0>();
  if (kCheck && bad) atomicOr(bad_flag, 1);
}

// =========================================================== phase B
// Forward pull recurrence.  kMarg: emit marginals e_k * exp2(M + beta - Z).
template <bool kMarg, bool kCheck>
__device__ void nw_forward(const float* __restrict__ th, int n, int m, int NW, const NwShared& sh,
                           const float* __restrict__ wsb, const float* __restrict__ wsk, float zint, float zfrac,
                           float* __restrict__ marg, float* last_v, float* last_o, int* bad_flag) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int j = 32 * w + l;
  const bool col_ok = j <= m;
  const int steps = n + 32;
  const int nblk = (steps + 1 + (NW - 1) * kLag + kP + kBlk - 1) / kBlk;
  const size_t rowstride = (size_t)(m + 1) * 3;
  float* ring_l = sh.ring + (size_t)w * kR * 96 + l;
  const uint32_t ring_u = smem_u32(sh.ring + (size_t)w * kR * 96) + 4u * l;
  const float* bq = sh.bq + (size_t)w * kRP * 32 + l;
  const float* bk = sh.bk + (size_t)w * kRP;
  const uint32_t bq_u = smem_u32(bq), bk_u = smem_u32(bk);
  const float2* bnd_in = sh.bnd0 + w * kRB;
  float2* bnd_out = sh.bnd0 + (w + 1) * kRB;
  const bool pub = (l == 31) & (w + 1 < NW);
  const bool zok = zfrac != ninf();
  bool bad = false;
  VO cur{ninf(), 0.f}, lprev{ninf(), 0.f};
  float av = ninf(), O = 0.f;  // own previous cell (i-1, j) in frame O
  const float* src_col = th + (size_t)(col_ok ? j : m) * 3;
  float* dst_col = kMarg ? marg + (size_t)(col_ok ? j : 0) * 3 : nullptr;
  const float* wsb_l = kMarg ? wsb + (size_t)w * steps * 32 + l : nullptr;
  const float* wsk_w = kMarg ? wsk + (size_t)w * steps : nullptr;
  for (int blk = 0; blk < nblk; ++blk) {
    const int s0 = -kP - w * kLag + blk * kBlk;
    if ((s0 + kBlk - 1 < -kP) | (s0 > steps)) {  // pipeline fill/drain: nothing to load or compute
      __syncthreads();
      continue;
    }
    const int pbase = mod_pos(s0 + kP, kR);
    const int cbase = mod_pos(s0 - l, kR);
    const int obase = mod_pos(s0 - 32, kR);
    const int q0 = s0 & (kRP - 1), qp = (s0 + kP) & (kRP - 1);  // multiples of kBlk: + k never wraps
    const int b0 = s0 & (kRB - 1);
    auto step = [&](auto steady_c, int k) {
      constexpr bool kS = decltype(steady_c)::value;
      const int s = s0 + k;
      {
        const int rp = s + kP;
        const bool pv = kS ? true : ((rp >= 0) & (rp <= n));
        const float* src = src_col + (size_t)(pv ? rp : 0) * rowstride;
        const uint32_t dst = ring_u + (uint32_t)(pbase + k) * 384u;
        cp4p(dst, src, pv);
        cp4p(dst + 128, src + 1, pv);
        cp4p(dst + 256, src + 2, pv);
        if (kMarg) {
          const bool bv = kS ? true : ((rp >= 0) & (rp < steps));
          const int rq = bv ? rp : 0;
          cp4p(bq_u + (uint32_t)(qp + k) * 128u, wsb_l + (size_t)rq * 32, bv);
          cp4p(bk_u + (uint32_t)(qp + k) * 4u, wsk_w + rq, bv & (l == 0));
        }
        cp_commit();
      }
      if (kS || (s >= 0 && s <= steps)) {
        cp_wait<kP>();
        if (kS || s < steps) {
          const int i = s - l;
          VO left;
          left.v = __shfl_up_sync(0xffffffffu, cur.v, 1);
          left.o = __shfl_up_sync(0xffffffffu, cur.o, 1);
          const bool inrow = kS ? true : ((i >= 0) & (i <= n));
          {
            const float2 a = bnd_in[b0 + k];
            const bool ok = (w > 0) & inrow;
            const bool l0 = l == 0;
            left.v = l0 ? (ok ? a.x : ninf()) : left.v;
            left.o = l0 ? (ok ? a.y : 0.f) : left.o;
          }
          const VO diag = lprev;
          lprev = left;
          const bool valid = inrow & col_ok;
          int cs = cbase + k;
          cs -= (cs >= kR) ? kR : 0;
          float* slot = ring_l + cs * 96;
          const float x0 = slot[0], x1 = slot[32], x2 = slot[64];
          if (kCheck) bad |= valid & (bad_input(x0) | bad_input(x1) | bad_input(x2));
          const float t0 = fmaf(x0, SDB_LOG2E, rel(diag, O));
          const float t1 = fmaf(x1, SDB_LOG2E, av);
          const float t2 = fmaf(x2, SDB_LOG2E, rel(left, O));
          const L3 r = lse3r(t0, t1, t2);
          const bool origin = kS ? false : ((i == 0) & (j == 0));
          if (kMarg) {
            const float bt = bq[(q0 + k) * 32];
            const float kk = bk[q0 + k];
            const float e = ex2((r.Mc + bt) + ((O + kk - zint) - zfrac));
            const float F = (zok & !origin) ? e : 0.f;
            slot[0] = r.e0 * F;
            slot[32] = r.e1 * F;
            slot[64] = r.e2 * F;
          }
          float a = origin ? 0.f : r.v;
          O = origin ? 0.f : O + r.r;
          a = valid ? a : ninf();
          av = a;
          if (!kS && valid && i == n && j == m) {
            *last_v = a;
            *last_o = O;
          }
          cur = VO{a, O};
          if (pub & inrow) bnd_out[i & (kRB - 1)] = make_float2(cur.v, cur.o);
        }
        if (kMarg) {
          const int r = s - 32;  // row completed by every lane of this warp
          if ((kS || ((r >= 0) & (r <= n))) & col_ok) {
            const float* slot = ring_l + (obase + k) * 96;
            float* dst = dst_col + (size_t)r * rowstride;
            dst[0] = slot[0];
            dst[1] = slot[32];
            dst[2] = slot[64];
          }
        }
      }
    };
    if (steady_block(s0, n)) {
#pragma unroll
      for (int k = 0; k < kBlk; ++k) step(BoolC<true>{}, k);
    } else {
#pragma unroll
      for (int k = 0; k < kBlk; ++k) step(BoolC<false>{}, k);
    }
    __syncthreads();
  }
  cp_wait<0>();
  if (kCheck && bad) atomicOr(bad_flag, 1);
}

__device__ void reset_prog(const NwShared& sh, int NW) {
  for (int q = threadIdx.x; q < NW; q += blockDim.x) sh.prog[q] = -kP - 1;
}

template <int kMode>  // 0 = logZ only, 1 = logZ + marginals
__global__ void nw_kernel(const float* __restrict__ theta, int n, int m, float* __restrict__ wsb_all,
                          float* __restrict__ wsk_all, double* __restrict__ logz, float* __restrict__ marg_all,
                          int32_t* __restrict__ status) {
  extern __shared__ __align__(16) char smraw[];
  __shared__ float zi, zf, lv, lo;
  __shared__ int badsh;
  const int NW = blockDim.x >> 5;
  const int b = blockIdx.x;
  NwShared sh = nw_carve(smraw, NW);
  const float* th = theta + (size_t)b * (n + 1) * (m + 1) * 3;
  const size_t wsz = (size_t)NW * (n + 32);
  if (threadIdx.x == 0) {
    zi = 0.f;
    zf = ninf();
    lv = ninf();
    lo = 0.f;
    badsh = 0;
  }
  reset_prog(sh, NW);
  __syncthreads();
  if (kMode == 1) {
    float* wsb = wsb_all + (size_t)b * wsz * 32;
    float* wsk = wsk_all + (size_t)b * wsz;
    nw_backward<true>(th, n, m, NW, sh, wsb, wsk, &zi, &zf, &badsh);
    __syncthreads();
    reset_prog(sh, NW);
    __syncthreads();
    nw_forward<true, false>(th, n, m, NW, sh, wsb, wsk, zi, zf, marg_all + (size_t)b * (n + 1) * (m + 1) * 3,
                            &lv, &lo, &badsh);
  } else {
    nw_forward<false, true>(th, n, m, NW, sh, nullptr, nullptr, 0.f, ninf(), nullptr, &lv, &lo, &badsh);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double z = (lv == ninf()) ? ninfd() : ((double)lo + (double)lv) * (double)SDB_LN2;
    status[b] = badsh ? SDB_ST_INVALID : (z == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
    logz[b] = z;
  }
}

// =========================================================== max-plus
// fp64 max-plus over the same skew with CTA barriers (argmax is not on the
// timed path); per-cell first-maximum choice in DIAG, DOWN, RIGHT order
// among in-grid sources (alignment.py:121-136, 153-167).
constexpr int kSyncM = 4;
constexpr int kLagM = 32 + kSyncM - 1;

__global__ void nw_max_kernel(const float* __restrict__ theta, int n, int m, int8_t* __restrict__ choice_all,
                              double* __restrict__ score, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) char smraw[];
  __shared__ double lastsh;
  __shared__ int badsh;
  const int NW = blockDim.x >> 5;
  const int b = blockIdx.x;
  NwShared sh = nw_carve(smraw, NW);
  double* bnd = reinterpret_cast<double*>(sh.bnd0);
  const float* th = theta + (size_t)b * (n + 1) * (m + 1) * 3;
  const int steps = n + 32;
  int8_t* choice = choice_all + (size_t)b * NW * steps * 32;
  if (threadIdx.x == 0) {
    lastsh = ninfd();
    badsh = 0;
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int j = 32 * w + l;
  const bool col_ok = j <= m;
  const int G = steps + (NW - 1) * kLagM;
  const size_t rowstride = (size_t)(m + 1) * 3;
  float* ring = sh.ring + (size_t)w * kR * 96;
  int bad = 0;
  double aprev = ninfd(), cur = ninfd(), lprev = ninfd();
  for (int g = -kP; g < G; ++g) {
    const int s = g - w * kLagM;
    {
      const int rp = s + kP;
      const bool pv = (rp >= 0) & (rp <= n) & col_ok;
      const float* src = th + (size_t)(pv ? rp : 0) * rowstride + (size_t)(col_ok ? j : 0) * 3;
      const uint32_t dst = smem_u32(ring + mod_pos(rp, kR) * 96 + l);
      cp4p(dst, src, pv);
      cp4p(dst + 128, src + 1, pv);
      cp4p(dst + 256, src + 2, pv);
      cp_commit();
    }
    if (s >= 0 && s < steps) {
      cp_wait<kP>();
      const int i = s - l;
      double left = __shfl_up_sync(0xffffffffu, cur, 1);
      if (l == 0) left = (w == 0 || i < 0 || i > n) ? ninfd() : bnd[w * kRB + (i & (kRB - 1))];
      const double diag = lprev;
      lprev = left;
      const bool valid = i >= 0 && i <= n && col_ok;
      double a = ninfd();
      if (valid) {
        const float* slot = ring + mod_pos(i, kR) * 96 + l;
        const float t0 = slot[0], t1 = slot[32], t2 = slot[64];
        bad |= bad_input(t0) | bad_input(t1) | bad_input(t2);
        const double c0 = diag + (double)t0, c1 = aprev + (double)t1, c2 = left + (double)t2;
        int k = 0;
        double best = ninfd();
        bool first = true;
        if (i > 0 && j > 0) { best = c0; k = 0; first = false; }
        if (i > 0 && (first || c1 > best)) { best = c1; k = 1; first = false; }
        if (j > 0 && (first || c2 > best)) { best = c2; k = 2; first = false; }
        a = (i == 0 && j == 0) ? 0.0 : best;
        choice[((size_t)w * steps + s) * 32 + l] = (int8_t)k;
        aprev = a;
        if (i == n && j == m) lastsh = a;
      }
      cur = valid ? a : ninfd();
      if (l == 31 && w + 1 < NW && i >= 0 && i <= n) bnd[(w + 1) * kRB + (i & (kRB - 1))] = cur;
    }
    if (((g + 1) % kSyncM) == 0) __syncthreads();
  }
  cp_wait<0>();
  if (bad) atomicOr(&badsh, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    const double z = lastsh;
    status[b] = badsh ? SDB_ST_INVALID : (z == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
    score[b] = z;
  }
}

// backtrack: one thread per instance walks the choices (strip layout) from
// (n, m) to (0, 0) and marks the path.
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

// =========================================================== meet in the middle
// Marginals with the forward and the backward recurrence running
// CONCURRENTLY in one CTA (warps [0,NW) forward strips, [NW,2NW) backward
// strips), each over half of the grid, then crossing over:
//   phase 1: forward computes alpha on A = {(i,j): i <= RF(strip(j))} and
//            stores it; backward computes beta on the complement B and stores
//            it.  RF(w) = (40 (NW-1-2w) + n - 1) / 2 balances the two so that
//            every strip of both directions finishes phase 1 in the same
//            block.  A is closed under predecessors, so every path crosses
//            from A to B exactly once and
//              Z = sum over crossing moves of alpha(src) e^theta(dst) beta(dst);
//   phase 2: forward continues on B emitting e_k * exp2(M + beta - Z) (as in
//            nw_forward), backward continues on A emitting
//            exp2(alpha(src_k) + theta_k + beta - Z) from the stored alpha.
// Both directions keep their own per-lane frames (values stored as (v, O)
// float2, exact).  Wall time is ~one wavefront pass instead of two, with twice
// the warps in flight.  Delay lines are split into two 16-lane halves
// (rows s-l for lanes 0-15 and 16-31 are 16 steps apart), which halves their
// shared memory so that two CTAs fit on an SM.
#ifndef SDB_MITM_BLK
#define SDB_MITM_BLK 8
#endif
constexpr int kMBlk = SDB_MITM_BLK;          // steps per barrier block
constexpr int kMLag = kMBlk == 4 ? 36 : kMBlk == 8 ? 40 : 48;  // >= 32 + kMBlk - 1, a multiple of kMBlk; kMLag + kMBlk < 96 (ring)
static_assert(kMLag >= 31 + kMBlk && kMLag % kMBlk == 0 && kMLag + kMBlk < 96 && kRB % kMBlk == 0, "mitm lag");
constexpr int kMP = 4;                       // potentials prefetch distance (steps)
constexpr int kMRh = 20;                     // delay-line rows per half-warp (>= 16 + kMP)
constexpr int kMGrp = kMRh * 48 + 16;        // floats per half-warp ring incl. 16-word bank pad
constexpr int kMRing = kMGrp + kMRh * 48;    // floats per warp
constexpr int kMS = 8;                       // alpha/beta slab ring entries (>= kMP + 2, power of 2)

struct MShared {
  float* ring;     // [2NW][kMRing]
  float2* bndF;    // [NW][kRB]  forward strip boundary
  float2* bndB0;   // [NW][kRB]  backward right push
  float2* bndB1;   // [NW][kRB]  backward diagonal push
  float2* slab;    // [2NW][kMS][32]
  float2* slabL;   // [NW][kMS]  backward: left-strip lane-31 alpha
  double* red;     // [64]
  int* flags;      // [4]
};

size_t mitm_smem_bytes(int NW) {
  return (size_t)2 * NW * kMRing * 4 + (size_t)3 * NW * kRB * 8 + (size_t)2 * NW * kMS * 32 * 8 +
         (size_t)NW * kMS * 8 + 64 * 8 + 16 + 64;
}

__device__ MShared mitm_carve(char* base, int NW) {
  MShared s;
  s.ring = (float*)base;
  base += (size_t)2 * NW * kMRing * 4;
  s.slab = (float2*)base;
  base += (size_t)2 * NW * kMS * 32 * 8;
  s.bndF = (float2*)base;
  base += (size_t)NW * kRB * 8;
  s.bndB0 = (float2*)base;
  base += (size_t)NW * kRB * 8;
  s.bndB1 = (float2*)base;
  base += (size_t)NW * kRB * 8;
  s.slabL = (float2*)base;
  base += (size_t)NW * kMS * 8;
  s.red = (double*)base;
  base += 64 * 8;
  s.flags = (int*)base;
  return s;
}

__device__ __forceinline__ int mitm_rf(int w, int n, int NW) { return (kMLag * (NW - 1 - 2 * w) + n - 1) >> 1; }
__device__ __forceinline__ int wrapr(int x) { return x >= kMRh ? x - kMRh : x; }
__device__ __forceinline__ void cp8p(uint32_t saddr, const void* gmem, bool pred) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p cp.async.ca.shared.global [%0], [%1], 8;\n}\n" ::"r"(saddr),
      "l"(gmem), "r"((int)pred));
}
__device__ __forceinline__ void bar_all() { asm volatile("bar.sync 0;\n" ::: "memory"); }
// per-direction barrier: forward warps use barrier 1, backward warps barrier 2
// (they only meet at the phase boundary)
__device__ __forceinline__ void bar_dir(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

template <int V>
struct IntC {
  static constexpr int value = V;
};

struct FState {
  VO cur, lprev;
  float av, O;
};
struct BState {
  VO pDn, pR, pD, savedD;
  float O;
};

// Blocks of one pass: s0 = -kMBlk - kMLag*w + kMBlk*(blk + off); consumption of
// row s-l by lane l at step s, exactly like nw_forward.
template <int kPh>
__device__ __forceinline__ void mitm_fwd(const float* __restrict__ th, int n, int m, int NW, const MShared& sh, int RF, int off,
                         int nblk, float2* __restrict__ wsa, const float2* __restrict__ wsb, float zint, float zfrac,
                         float* __restrict__ marg, FState& st, int* bad_flag, bool edge) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int g = l >> 4, q = l & 15;
  const int j = 32 * w + l;
  const bool col_ok = j < (edge ? m : m + 1);
  const bool lastcol = edge & (j == m - 1);  // alpha(., m-1) is kept for every row (edge column epilogue)
  const int steps = n + 32;
  const int lo = kPh == 1 ? 0 : RF + 1, hi = kPh == 1 ? RF : n;
  const size_t rowstride = (size_t)(m + 1) * 3;
  float* ring_g = sh.ring + (size_t)w * kMRing + g * kMGrp + q;
  const uint32_t ring_u = smem_u32(ring_g);
  const float* src_col = th + (size_t)(col_ok ? j : m) * 3;
  float* dst_col = kPh == 2 ? marg + (size_t)(col_ok ? j : 0) * 3 : nullptr;
  float2* wsa_l = wsa + (size_t)w * steps * 32 + l;
  const float2* wsb_l = wsb + (size_t)w * steps * 32 + l;
  float2* slab_w = sh.slab + (size_t)w * kMS * 32;
  const uint32_t slab_u = smem_u32(slab_w + l);
  const float2* bnd_in = sh.bndF + w * kRB;
  float2* bnd_out = sh.bndF + (w + 1) * kRB;
  const bool pub = (l == 31) & (w + 1 < NW);
  const bool zok = zfrac != ninf();
  const int s_lo = max(lo, 1) + 32, s_hi = min(hi, n - 1) - (kMBlk - 1) - kMP;
  bool bad = false;
  VO cur = st.cur, lprev = st.lprev;
  float av = st.av, O = st.O;
  for (int blk = 0; blk < nblk; ++blk) {
    const int s0 = -kMBlk - w * kMLag + (blk + off) * kMBlk;
    if ((s0 + kMBlk - 1 + kMP < max(lo, 0)) | (s0 > hi + 32 + (kPh == 2 ? 1 : 0))) {
      bar_dir(1, 32 * NW);
      continue;
    }
    const int pb = mod_pos(s0 + kMP - 16 * g, kMRh);
    const int cb = mod_pos(s0 - l, kMRh);
    const int wb = mod_pos(s0 - 16 - 16 * g, kMRh);
    const int b0 = s0 & (kRB - 1);
    const ptrdiff_t rs = (ptrdiff_t)rowstride;
    const float* tsrc = src_col + (ptrdiff_t)(s0 + kMP - 16 * g) * rs;  // advanced one row per step
    float* wdst = kPh == 2 ? dst_col + (ptrdiff_t)(s0 - 16 - 16 * g) * rs : nullptr;
    float2* wsa_b = wsa_l + (ptrdiff_t)s0 * 32;
    const float2* wsb_b = wsb_l + (ptrdiff_t)(s0 + kMP) * 32;
    auto step = [&](auto steady_c, int k) {
      // mode 1 = steady (every lane active, interior of the grid), 2 = interior
      // (grid-edge cases impossible, lanes straddle the phase boundary), 0 = generic
      constexpr int kMode = decltype(steady_c)::value;
      constexpr bool kS = kMode == 1, kIn = kMode >= 1;
      const int s = s0 + k;
      if (kPh == 2) {  // write back the row this half-warp completed at step s-1 (before its slot is refilled)
        const int r = s - 16 - 16 * g;
        if ((kS || ((r >= lo) & (r <= hi))) & col_ok) {
          const float* slot = ring_g + wrapr(wb + k) * 48;
          wdst[0] = slot[0];
          wdst[1] = slot[16];
          wdst[2] = slot[32];
        }
        wdst += rs;
      }
      {
        const int prow = s + kMP - 16 * g;
        const bool pv = kIn ? true : ((prow >= 0) & (prow <= n));
        const float* src = tsrc;
        tsrc += rs;
        const uint32_t dst = ring_u + (uint32_t)wrapr(pb + k) * 192u;
        cp4p(dst, src, pv);
        cp4p(dst + 64, src + 1, pv);
        cp4p(dst + 128, src + 2, pv);
        if (kPh == 2) {
          const int sp = s + kMP;
          const bool bv = kIn ? true : ((sp >= 0) & (sp < steps));
          cp8p(slab_u + (uint32_t)((s + kMP) & (kMS - 1)) * 256u, wsb_b + 32 * k, bv);
        }
        cp_commit();
      }
      if (kIn || ((s >= 0) & (s < steps))) {
        cp_wait<kMP>();
        const int i = s - l;
        VO left;
        left.v = __shfl_up_sync(0xffffffffu, cur.v, 1);
        left.o = __shfl_up_sync(0xffffffffu, cur.o, 1);
        const bool inrow = kIn ? true : ((i >= 0) & (i <= n));
        {
          const float2 a = bnd_in[b0 + k];
          const bool ok = (w > 0) & inrow;
          const bool l0 = l == 0;
          left.v = l0 ? (ok ? a.x : ninf()) : left.v;
          left.o = l0 ? (ok ? a.y : 0.f) : left.o;
        }
        const bool act = kS ? true : ((i >= lo) & (i <= hi) & col_ok);
        float* slot = ring_g + wrapr(cb + k) * 48;
        const float x0 = slot[0], x1 = slot[16], x2 = slot[32];
        bad |= act & col_ok & (bad_input(x0) | bad_input(x1) | bad_input(x2));
        const float t0 = fmaf(x0, SDB_LOG2E, rel(lprev, O));
        const float t1 = fmaf(x1, SDB_LOG2E, av);
        const float t2 = fmaf(x2, SDB_LOG2E, rel(left, O));
        const L3 r = lse3r(t0, t1, t2);
        const bool origin = kIn ? false : ((i == 0) & (j == 0));
        if (kPh == 2) {
          const float2 bt = slab_w[(s & (kMS - 1)) * 32 + l];
          const float e = ex2((r.Mc + bt.x) + ((O + bt.y - zint) - zfrac));
          const float F = (zok & act) ? e : 0.f;
          slot[0] = r.e0 * F;
          slot[16] = r.e1 * F;
          slot[32] = r.e2 * F;
        }
        const float a = origin ? 0.f : r.v;
        const float On = origin ? 0.f : O + r.r;
        if (kS) {
          lprev = left;
          av = a;
          O = On;
          cur = VO{a, On};
        } else if (act) {
          lprev = left;
          av = a;
          O = On;
          cur = VO{a, On};
        }
        if ((kPh == 1 || lastcol) && (kS || act)) wsa_b[32 * k] = make_float2(a, On);
        if (pub & (kS || act)) bnd_out[i & (kRB - 1)] = make_float2(a, On);
      }
    };
    if ((s0 >= s_lo) & (s0 <= s_hi)) {
#pragma unroll
      for (int k = 0; k < kMBlk; ++k) step(IntC<1>{}, k);
    } else if ((s0 >= 32) & (s0 + kMBlk - 1 + kMP <= n - 1)) {
#pragma unroll 1
      for (int k = 0; k < kMBlk; ++k) step(IntC<2>{}, k);
    } else {
#pragma unroll 1
      for (int k = 0; k < kMBlk; ++k) step(IntC<0>{}, k);
    }
    bar_dir(1, 32 * NW);
  }
  cp_wait<0>();
  st.cur = cur;
  st.lprev = lprev;
  st.av = av;
  st.O = O;
  if (bad) atomicOr(bad_flag, 1);
}

// Backward strips on the flipped grid (as nw_backward).  Warp wb = warp - NW
// handles flipped columns jo = 32 NW - 1 - (32 wb + l), i.e. original strip
// u = NW-1-wb with forward lane 31-l.
template <int kPh>
__device__ __forceinline__ void mitm_bwd(const float* __restrict__ th, int n, int m, int NW, const MShared& sh, int RFu, int off,
                         int nblk, const float2* __restrict__ wsa, float2* __restrict__ wsb, float zint, float zfrac,
                         float* __restrict__ marg, BState& st, bool edge, const float2* __restrict__ pushR,
                         const float2* __restrict__ pushD) {
  const int wb = (threadIdx.x >> 5) - NW, l = threadIdx.x & 31;
  const int g = l >> 4, q = l & 15;
  const int mp = 32 * NW - 1;
  const int jo = mp - (32 * wb + l);
  const bool col_ok = jo < (edge ? m : m + 1);
  // edge mode: column m is not in a strip; lane 0 of warp 0 (column m-1) streams
  // that column's pushes (precomputed by mitm_edge_prologue) into warp 0's
  // otherwise unused boundary rings
  const bool edge_lane = edge & (wb == 0) & (l == 0);
  const uint32_t e0_u = smem_u32(sh.bndB0), e1_u = smem_u32(sh.bndB1);
  const int u = NW - 1 - wb, lf = 31 - l;
  const int steps = n + 32;
  const int QB = n - RFu - 1;  // flipped rows [0, QB] are original rows > RF(u)
  const int lo = kPh == 1 ? 0 : QB + 1, hi = kPh == 1 ? QB : n;
  const size_t rowstride = (size_t)(m + 1) * 3;
  float* ring_g = sh.ring + (size_t)(NW + wb) * kMRing + g * kMGrp + q;
  const uint32_t ring_u = smem_u32(ring_g);
  const float* src_col = th + (size_t)(col_ok ? jo : m) * 3;
  float* dst_col = kPh == 2 ? marg + (size_t)(col_ok ? jo : 0) * 3 : nullptr;
  float2* wsb_l = wsb + (size_t)u * steps * 32 + lf;
  const float2* wsa_u = wsa + (size_t)u * steps * 32;
  const float2* wsa_left = u > 0 ? wsa + (size_t)(u - 1) * steps * 32 + 31 : nullptr;
  float2* slab_w = sh.slab + (size_t)(NW + wb) * kMS * 32;
  const uint32_t slab_u = smem_u32(slab_w + l);
  float2* slabL = sh.slabL + wb * kMS;
  const uint32_t slabL_u = smem_u32(slabL);
  const float2* bnd0_in = sh.bndB0 + wb * kRB;
  const float2* bnd1_in = sh.bndB1 + wb * kRB;
  float2* bnd0_out = sh.bndB0 + (wb + 1) * kRB;
  float2* bnd1_out = sh.bndB1 + (wb + 1) * kRB;
  const bool pub = (l == 31) & (wb + 1 < NW);
  const bool zok = zfrac != ninf();
  const int s_lo = max(lo, 1) + 32, s_hi = min(hi, n - 1) - (kMBlk - 1) - kMP;
  VO pDn = st.pDn, pR = st.pR, pD = st.pD, savedD = st.savedD;
  float O = st.O;
  float2 c1 = make_float2(ninf(), 0.f), c2 = make_float2(ninf(), 0.f);  // phase 2 alpha carries
  for (int blk = 0; blk < nblk; ++blk) {
    const int s0 = -kMBlk - wb * kMLag + (blk + off) * kMBlk;
    if ((s0 + kMBlk - 1 + kMP < max(lo, 0)) | (s0 > hi + 32 + (kPh == 2 ? 1 : 0))) {
      bar_dir(2, 32 * NW);
      continue;
    }
    const int pb = mod_pos(s0 + kMP - 16 * g, kMRh);
    const int cb = mod_pos(s0 - l, kMRh);
    const int wbk = mod_pos(s0 - 16 - 16 * g, kMRh);
    const int b0 = s0 & (kRB - 1);
    const ptrdiff_t rs = (ptrdiff_t)rowstride;
    const float* tsrc = src_col + (ptrdiff_t)(n - (s0 + kMP - 16 * g)) * rs;  // moves up one row per step
    float* wdst = kPh == 2 ? dst_col + (ptrdiff_t)(n - (s0 - 16 - 16 * g)) * rs : nullptr;
    float2* wsb_b = wsb_l + (ptrdiff_t)(n + 31 - s0) * 32;
    const float2* sa_b = wsa_u + (ptrdiff_t)(n + 29 - kMP - s0) * 32 + l;
    const float2* sl_b = u > 0 ? wsa_left + (ptrdiff_t)(n + 29 - kMP + 32 - s0) * 32 : wsa_u;
    auto step = [&](auto steady_c, int k) {
      // mode 1 = steady (every lane active, interior of the grid), 2 = interior
      // (grid-edge cases impossible, lanes straddle the phase boundary), 0 = generic
      constexpr int kMode = decltype(steady_c)::value;
      constexpr bool kS = kMode == 1, kIn = kMode >= 1;
      const int s = s0 + k;
      if (kPh == 2) {
        const int r = s - 16 - 16 * g;  // flipped row completed at step s-1
        if ((kS || ((r >= lo) & (r <= hi))) & col_ok) {
          const float* slot = ring_g + wrapr(wbk + k) * 48;
          wdst[0] = slot[0];
          wdst[1] = slot[16];
          wdst[2] = slot[32];
        }
        wdst -= rs;
      }
      {
        const int prow = s + kMP - 16 * g;
        const bool pv = kIn ? true : ((prow >= 0) & (prow <= n));
        const float* src = tsrc;
        tsrc -= rs;
        const uint32_t dst = ring_u + (uint32_t)wrapr(pb + k) * 192u;
        cp4p(dst, src, pv);
        cp4p(dst + 64, src + 1, pv);
        cp4p(dst + 128, src + 2, pv);
        if (kPh == 2) {
          // alpha slab sF(s+kMP)-2 (own strip) and left-strip lane-31 alpha for sF(s+kMP)-1
          const int sa = n + 29 - s - kMP;
          const bool av_ = kIn ? true : ((sa >= 0) & (sa < steps));
          cp8p(slab_u + (uint32_t)(sa & (kMS - 1)) * 256u, sa_b - 32 * k, av_);
          const int sl = sa + 1 + 31;
          const bool lv = (u > 0) & (l == 0) & (sl >= 0) & (sl < steps);
          cp8p(slabL_u + (uint32_t)((sa + 1) & (kMS - 1)) * 8u, sl_b - 32 * k, lv);
        }
        {
          const int sp = s + kMP;
          const bool ev = edge_lane & (kIn ? true : ((sp >= 0) & (sp <= n)));
          cp8p(e0_u + (uint32_t)(sp & (kRB - 1)) * 8u, pushR + sp, ev);
          cp8p(e1_u + (uint32_t)(sp & (kRB - 1)) * 8u, pushD + sp, ev);
        }
        cp_commit();
      }
      if (kIn || ((s >= 0) & (s < steps))) {
        cp_wait<kMP>();
        const int ip = s - l;
        VO rR, rD;
        rR.v = __shfl_up_sync(0xffffffffu, pR.v, 1);
        rR.o = __shfl_up_sync(0xffffffffu, pR.o, 1);
        rD.v = __shfl_up_sync(0xffffffffu, pD.v, 1);
        rD.o = __shfl_up_sync(0xffffffffu, pD.o, 1);
        const bool inrow = kIn ? true : ((ip >= 0) & (ip <= n));
        {
          const float2 a = bnd0_in[b0 + k], d = bnd1_in[b0 + k];
          const bool ok = ((wb > 0) | edge) & inrow;
          const bool l0 = l == 0;
          rR.v = l0 ? (ok ? a.x : ninf()) : rR.v;
          rR.o = l0 ? (ok ? a.y : 0.f) : rR.o;
          rD.v = l0 ? (ok ? d.x : ninf()) : rD.v;
          rD.o = l0 ? (ok ? d.y : 0.f) : rD.o;
        }
        const bool act = kS ? true : ((ip >= lo) & (ip <= hi) & col_ok);
        float* slot = ring_g + wrapr(cb + k) * 48;
        const float x0 = slot[0], x1 = slot[16], x2 = slot[32];
        const L3 r = lse3r(rel(savedD, O), rel(pDn, O), rel(rR, O));
        float b, On;
        if (kIn) {
          b = r.v;
          On = O + r.r;
        } else {
          const bool start = (ip == 0) & (jo == m);
          b = start ? 0.f : r.v;
          On = start ? 0.f : O + r.r;
        }
        if (kPh == 2) {
          // original cell (i, j) = (n - ip, jo); alpha of its three sources.  One slab
          // entry per step: X = alpha(i-1, j) of the NEXT step's cell; the left column
          // comes from lane l+1 (lf-1) or, for lf = 0, from the left strip's lane 31.
          // alpha(i-1, j) and alpha(i, j-1) are the previous step's X and left value.
          __syncwarp();
          const int sF = n + 31 - s;
          const int i = n - ip;
          const float2 X = slab_w[((sF - 2) & (kMS - 1)) * 32 + lf];
          float2 Y;
          Y.x = __shfl_down_sync(0xffffffffu, X.x, 1);
          Y.y = __shfl_down_sync(0xffffffffu, X.y, 1);
          {
            const float2 L = slabL[(sF - 1) & (kMS - 1)];
            Y.x = l == 31 ? L.x : Y.x;
            Y.y = l == 31 ? L.y : Y.y;
          }
          const float2 A0 = Y, A1 = c1, A2 = c2;
          c1 = X;
          c2 = Y;
          const bool hi_ok = kIn ? true : (i >= 1), left_ok = jo >= 1, ok = kS ? zok : (zok & act);
          const float base = b - zfrac;
          const float e0 = ex2(((A0.y + On - zint) + (A0.x + fmaf(x0, SDB_LOG2E, base))));
          const float e1 = ex2(((A1.y + On - zint) + (A1.x + fmaf(x1, SDB_LOG2E, base))));
          const float e2 = ex2(((A2.y + On - zint) + (A2.x + fmaf(x2, SDB_LOG2E, base))));
          slot[0] = (ok & hi_ok & left_ok) ? e0 : 0.f;
          slot[16] = (ok & hi_ok) ? e1 : 0.f;
          slot[32] = (ok & left_ok) ? e2 : 0.f;
        }
        // invalid (padding) columns push -inf with offset 0 so they never poison real lanes
        const bool okb = kS ? col_ok : act;
        const float bb = okb ? b : ninf();
        if (kS && !col_ok) On = 0.f;
        const VO nD{fmaf(x0, SDB_LOG2E, bb), On}, nDn{fmaf(x1, SDB_LOG2E, bb), On}, nR{fmaf(x2, SDB_LOG2E, bb), On};
        if (kS) {
          savedD = rD;
          pD = nD;
          pDn = nDn;
          pR = nR;
          O = On;
        } else if (act) {
          savedD = rD;
          pD = nD;
          pDn = nDn;
          pR = nR;
          O = On;
        }
        if (kPh == 1 && (kS || act)) wsb_b[-32 * k] = make_float2(b, On);
        if (pub & (kS || act)) {
          bnd0_out[ip & (kRB - 1)] = make_float2(nR.v, nR.o);
          bnd1_out[ip & (kRB - 1)] = make_float2(nD.v, nD.o);
        }
      }
    };
    if ((s0 >= s_lo) & (s0 <= s_hi)) {
#pragma unroll
      for (int k = 0; k < kMBlk; ++k) step(IntC<1>{}, k);
    } else if ((s0 >= 32) & (s0 + kMBlk - 1 + kMP <= n - 1)) {
#pragma unroll 1
      for (int k = 0; k < kMBlk; ++k) step(IntC<2>{}, k);
    } else {
#pragma unroll 1
      for (int k = 0; k < kMBlk; ++k) step(IntC<0>{}, k);
    }
    bar_dir(2, 32 * NW);
  }
  cp_wait<0>();
  st.pDn = pDn;
  st.pR = pR;
  st.pD = pD;
  st.savedD = savedD;
  st.O = O;
}

// log2 Z over the moves that cross from A into B (fp64, all threads).  In
// edge mode column m is entirely in B: its entry moves from column m-1 (DIAG
// into rows 1..RF(NW-1)+1, RIGHT into rows 0..RF(NW-1)) are crossings too.
__device__ double mitm_z(const float* __restrict__ th, int n, int m, int NW, const float2* __restrict__ wsa,
                         const float2* __restrict__ wsb, double* red, bool edge, const double* __restrict__ betaM) {
  const int steps = n + 32;
  const int m1 = m + 1;
  const int mc = edge ? m : m1;  // strip columns
  const int RFl = mitm_rf(NW - 1, n, NW);
  // per column: DOWN and DIAG into row RF+1; per strip boundary 32w: RIGHT into
  // rows (RF(w), RF(w-1)] and DIAG into rows (RF(w)+1, RF(w-1)+1]
  const int Eb = 2 * mc + 2 * (mitm_rf(0, n, NW) - RFl);
  const int E = Eb + (edge ? 2 * (RFl + 1) : 0);
  auto alpha = [&](int i, int j) {
    const float2 v = wsa[((size_t)(j >> 5) * steps + i + (j & 31)) * 32 + (j & 31)];
    return (double)v.x + (double)v.y;
  };
  auto beta = [&](int i, int j) {
    const float2 v = wsb[((size_t)(j >> 5) * steps + i + (j & 31)) * 32 + (j & 31)];
    return (double)v.x + (double)v.y;
  };
  auto theta = [&](int i, int j, int k) { return (double)th[((size_t)i * m1 + j) * 3 + k] * 1.4426950408889634; };
  double mx = ninfd(), sm = 0.0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    double t = ninfd();
    if (e >= Eb) {
      const int x = e - Eb;
      if (x <= RFl)  // RIGHT (x, m-1) -> (x, m)
        t = alpha(x, m - 1) + theta(x, m, 2) + betaM[x];
      else  // DIAG (i-1, m-1) -> (i, m), i = x - RFl
        t = alpha(x - RFl - 1, m - 1) + theta(x - RFl, m, 0) + betaM[x - RFl];
    } else if (e < 2 * mc) {
      const int j = e < mc ? e : e - mc;
      const int R = mitm_rf(j >> 5, n, NW);
      if (e < mc)
        t = alpha(R, j) + theta(R + 1, j, 1) + beta(R + 1, j);
      else if (j >= 1)
        t = alpha(R, j - 1) + theta(R + 1, j, 0) + beta(R + 1, j);
    } else {
      int x = e - 2 * mc, w = 1;
      while (x >= 2 * (mitm_rf(w - 1, n, NW) - mitm_rf(w, n, NW))) {
        x -= 2 * (mitm_rf(w - 1, n, NW) - mitm_rf(w, n, NW));
        ++w;
      }
      const int c = mitm_rf(w - 1, n, NW) - mitm_rf(w, n, NW), j = 32 * w;
      if (x < c) {
        const int i = mitm_rf(w, n, NW) + 1 + x;
        t = alpha(i, j - 1) + theta(i, j, 2) + beta(i, j);
      } else {
        const int i = mitm_rf(w, n, NW) + 2 + (x - c);
        t = alpha(i - 1, j - 1) + theta(i, j, 0) + beta(i, j);
      }
    }
    if (t != t) t = ninfd();
    if (t > mx) {
      sm = (mx == ninfd()) ? 1.0 : sm * exp2(mx - t) + 1.0;
      mx = t;
    } else if (t != ninfd()) {
      sm += exp2(t - mx);
    }
  }
  const int wi = threadIdx.x >> 5, li = threadIdx.x & 31, nw = blockDim.x >> 5;
  double gm = warp_maxd(mx);
  double gs = (mx == ninfd()) ? 0.0 : sm * exp2(mx - gm);
  for (int o = 16; o > 0; o >>= 1) gs += __shfl_xor_sync(0xffffffffu, gs, o);
  if (li == 0) {
    red[wi] = gm;
    red[32 + wi] = gs;
  }
  bar_all();
  double M = ninfd();
  for (int x = 0; x < nw; ++x) M = fmax(M, red[x]);
  double S = 0.0;
  if (M != ninfd())
    for (int x = 0; x < nw; ++x) S += (red[x] == ninfd()) ? 0.0 : red[32 + x] * exp2(red[x] - M);
  bar_all();
  return (M == ninfd()) ? ninfd() : M + log2(S);
}

// Edge mode (m % 32 == 0): the last column m would be a strip of its own with
// one live lane per direction.  It is not needed as one: every path that enters
// column m only moves DOWN afterwards, so
//   beta(i, m) = sum_{r > i} theta[r, m, DOWN]            (a suffix sum)
// and, with e(r) the marginal of the DIAG + RIGHT moves into (r, m),
//   p(DOWN into (i, m)) = sum_{r < i} e(r)                 (a prefix sum).
// The backward pass consumes column m's pushes from these sums, the forward
// pass never computes column m (alignment.py:62-118 define the same numbers
// through the full recurrences).
//
// Chunked block-wide scans in fp64: thread t owns rows [t*C, t*C + C).
__device__ double block_excl(double v, double* scratch, int t, int T, bool suffix, int bar_id) {
  scratch[t] = v;
  bar_dir(bar_id, T);
  double acc = 0.0;
  if (suffix)
    for (int x = t + 1; x < T; ++x) acc += scratch[x];
  else
    for (int x = 0; x < t; ++x) acc += scratch[x];
  bar_dir(bar_id, T);
  return acc;
}

// backward warps (T = 32 NW threads, barrier 2): betaM[i] = beta(i, m) (log2),
// pushR/pushD[ip] = the RIGHT / DIAG pushes of cell (n - ip, m) as (v, O).
__device__ void mitm_edge_prologue(const float* __restrict__ th, int n, int m, int NW, double* __restrict__ betaM,
                                   float2* __restrict__ pushR, float2* __restrict__ pushD, double* scratch,
                                   int* bad_flag) {
  const int T = 32 * NW, t = threadIdx.x - T;
  const int C = (n + 1 + T - 1) / T, r0 = min(t * C, n + 1), r1 = min(r0 + C, n + 1);
  const size_t rs = (size_t)(m + 1) * 3;
  const float* col = th + (size_t)m * 3;
  const double L = 1.4426950408889634;
  double cs = 0.0;
  bool bad = false;
  for (int r = r0; r < r1; ++r) {
    const float x0 = col[r * rs], x1 = col[r * rs + 1], x2 = col[r * rs + 2];
    bad |= bad_input(x0) | bad_input(x1) | bad_input(x2);
    if (r >= 1) cs += (double)x1 * L;
  }
  double b = block_excl(cs, scratch, t, T, true, 2);  // beta(r1 - 1, m)
  auto split = [](double x) {
    if (!(x > -1e300)) return make_float2(ninf(), 0.f);
    const double o = rint(x);
    return make_float2((float)(x - o), (float)o);
  };
  for (int r = r1 - 1; r >= r0; --r) {
    betaM[r] = b;
    pushR[n - r] = split((double)col[r * rs + 2] * L + b);
    pushD[n - r] = split((double)col[r * rs] * L + b);
    if (r >= 1) b += (double)col[r * rs + 1] * L;
  }
  if (bad) atomicOr(bad_flag, 1);
}

// all threads, after phase 2: column m's move marginals.
__device__ void mitm_edge_epilogue(const float* __restrict__ th, int n, int m, int NW, const float2* __restrict__ wsa,
                                   const double* __restrict__ betaM, double z2, float* __restrict__ marg,
                                   double* scratch) {
  const int T = blockDim.x, t = threadIdx.x;
  const int C = (n + 1 + T - 1) / T, r0 = min(t * C, n + 1), r1 = min(r0 + C, n + 1);
  const int steps = n + 32;
  const size_t rs = (size_t)(m + 1) * 3;
  const float* col = th + (size_t)m * 3;
  float* mc = marg + (size_t)m * 3;
  const double L = 1.4426950408889634;
  const bool zok = z2 != ninfd();
  const float2* wl = wsa + ((size_t)(NW - 1) * steps + 31) * 32 + 31;  // alpha(i, m-1) at wl[32 i]
  auto alpha = [&](int i) { const float2 v = wl[(size_t)i * 32]; return (double)v.x + (double)v.y; };
  auto entry = [&](int r, double& ed, double& er) {
    ed = (zok & (r >= 1)) ? exp2(alpha(r - 1) + (double)col[r * rs] * L + betaM[r] - z2) : 0.0;
    er = zok ? exp2(alpha(r) + (double)col[r * rs + 2] * L + betaM[r] - z2) : 0.0;
  };
  double cs = 0.0;
  for (int r = r0; r < r1; ++r) {
    double ed, er;
    entry(r, ed, er);
    mc[r * rs] = (float)ed;
    mc[r * rs + 2] = (float)er;
    cs += ed + er;
  }
  double run = block_excl(cs, scratch, t, T, false, 0);
  for (int r = r0; r < r1; ++r) {
    double ed, er;
    entry(r, ed, er);
    mc[r * rs + 1] = (float)run;  // 0 for r = 0
    run += ed + er;
  }
}

// kMaxT = 640 for NW >= 9: 18-20 warps put 5 on one SM sub-partition, whose
// 16K registers then cap the kernel at 96 registers per thread.
template <int kMaxT>
__global__ void __launch_bounds__(kMaxT) nw_mitm_kernel(const float* __restrict__ theta, int n, int m, float2* __restrict__ wsa_all,
                               float2* __restrict__ wsb_all, double* __restrict__ edge_all, double* __restrict__ logz,
                               float* __restrict__ marg_all, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) char smraw[];
  const int NW = blockDim.x >> 6;
  const int b = blockIdx.x;
  MShared sh = mitm_carve(smraw, NW);
  const float* th = theta + (size_t)b * (n + 1) * (m + 1) * 3;
  float* marg = marg_all + (size_t)b * (n + 1) * (m + 1) * 3;
  const size_t wsz = (size_t)NW * (n + 32) * 32;
  float2* wsa = wsa_all + (size_t)b * wsz;
  float2* wsb = wsb_all + (size_t)b * wsz;
  const bool edge = (m & 31) == 0;
  double* betaM = edge_all + (size_t)b * 3 * (n + 1);  // [n+1] doubles, then pushR, pushD [n+1] float2
  float2* pushR = (float2*)(betaM + (n + 1));
  float2* pushD = pushR + (n + 1);
  if (threadIdx.x == 0) sh.flags[0] = 0;
  const int warp = threadIdx.x >> 5;
  const bool fwd = warp < NW;
  const int w = fwd ? warp : warp - NW;
  // phase lengths (identical for every warp: one barrier per block)
  int G1 = 0, off2 = 1 << 30, G2 = 0;
  for (int x = 0; x < NW; ++x) {
    const int RF = mitm_rf(x, n, NW), QB = n - mitm_rf(NW - 1 - x, n, NW) - 1;
    G1 = max(G1, max((RF + 31 + kMBlk + kMLag * x) / kMBlk, (QB + 31 + kMBlk + kMLag * x) / kMBlk) + 1);
    off2 = min(off2, min((RF + 1 + kMLag * x) / kMBlk, (QB + 1 + kMLag * x) / kMBlk));
  }
  for (int x = 0; x < NW; ++x) G2 = max(G2, (n + 33 + kMBlk + kMLag * x) / kMBlk - off2 + 1);
  FState fs{{ninf(), 0.f}, {ninf(), 0.f}, ninf(), 0.f};
  BState bs{{ninf(), 0.f}, {ninf(), 0.f}, {ninf(), 0.f}, {ninf(), 0.f}, 0.f};
  bar_all();
  if (fwd) {
    mitm_fwd<1>(th, n, m, NW, sh, mitm_rf(w, n, NW), 0, G1, wsa, wsb, 0.f, ninf(), nullptr, fs, sh.flags, edge);
  } else {
    // the backward rings are free until the first prefetch: scratch for the scan
    if (edge) mitm_edge_prologue(th, n, m, NW, betaM, pushR, pushD, (double*)(sh.ring + (size_t)NW * kMRing), sh.flags);
    mitm_bwd<1>(th, n, m, NW, sh, mitm_rf(NW - 1 - w, n, NW), 0, G1, wsa, wsb, 0.f, ninf(), nullptr, bs, edge, pushR,
                pushD);
  }
  __threadfence_block();
  bar_all();
  const double z2 = mitm_z(th, n, m, NW, wsa, wsb, sh.red, edge, betaM);
  const float zint = (z2 == ninfd()) ? 0.f : (float)rint(z2);
  const float zfrac = (z2 == ninfd()) ? ninf() : (float)(z2 - rint(z2));
  if (fwd)
    mitm_fwd<2>(th, n, m, NW, sh, mitm_rf(w, n, NW), off2, G2, wsa, wsb, zint, zfrac, marg, fs, sh.flags, edge);
  else
    mitm_bwd<2>(th, n, m, NW, sh, mitm_rf(NW - 1 - w, n, NW), off2, G2, wsa, wsb, zint, zfrac, marg, bs, edge, pushR,
                pushD);
  __threadfence_block();
  bar_all();
  if (edge) mitm_edge_epilogue(th, n, m, NW, wsa, betaM, z2, marg, (double*)sh.ring);
  if (threadIdx.x == 0) {
    const double z = (z2 == ninfd()) ? ninfd() : z2 * (double)SDB_LN2;
    status[b] = sh.flags[0] ? SDB_ST_INVALID : (z == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
    logz[b] = z;
  }
}

// strips per direction: columns 0..m, or 0..m-1 when column m is an edge column
int mitm_nw(int m) { return (m & 31) == 0 ? m / 32 : (m + 1 + 31) / 32; }

int mitm_ok(int n, int m) {
  const int NW = mitm_nw(m);
  return NW <= 10 && n >= kMLag * (NW - 1) + 32 && mitm_smem_bytes(NW) <= 220 * 1024;
}

struct NwWs {
  float* wsb;
  float* wsk;
  int8_t* choice;
  float2* wsa2;  // meet-in-the-middle alpha / beta (v, O)
  float2* wsb2;
  double* edge;  // [B][3 (n+1)]: beta(., m) fp64, then the column-m pushes (edge mode)
};

NwWs nw_carve_ws(void* base, int64_t B, int n, int m, int mode, size_t* bytes) {
  const int NW = (m + 1 + 31) / 32;
  const size_t wsz = (size_t)NW * (n + 32);
  Carve c(base);
  NwWs w{};
  if (mode == 1 && mitm_ok(n, m)) {
    const size_t wsm = (size_t)mitm_nw(m) * (n + 32);
    w.wsa2 = c.take<float2>((size_t)B * wsm * 32);
    w.wsb2 = c.take<float2>((size_t)B * wsm * 32);
    w.edge = c.take<double>((m & 31) == 0 ? (size_t)B * 3 * (n + 1) : 1);
  } else if (mode == 1) {
    w.wsb = c.take<float>((size_t)B * wsz * 32);
    w.wsk = c.take<float>((size_t)B * wsz);
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
  if (kMode == 2) {
    if (sdb_set_smem((const void*)nw_max_kernel, smem) != cudaSuccess)
      return SDB_ERR_CUDA;
    nw_max_kernel<<<(unsigned)B, 32 * NW, smem, s>>>(theta, n, m, ws.choice, score, status);
    SDB_CHECK_LAUNCH();
    nw_walk_kernel<<<(unsigned)((B + 127) / 128), 128, 0, s>>>(ws.choice, n, m, NW, B, status, path);
    SDB_CHECK_LAUNCH();
    return SDB_OK;
  }
  if (kMode == 1 && ws.wsa2) {
    const int NWm = mitm_nw(m);
    const size_t sm2 = mitm_smem_bytes(NWm);
    auto kern = NWm >= 9 ? nw_mitm_kernel<640> : nw_mitm_kernel<512>;
    if (sdb_set_smem((const void*)kern, sm2) != cudaSuccess)
      return SDB_ERR_CUDA;
    kern<<<(unsigned)B, 64 * NWm, sm2, s>>>(theta, n, m, ws.wsa2, ws.wsb2, ws.edge, logz, marg, status);
    SDB_CHECK_LAUNCH();
    return SDB_OK;
  }
  constexpr int M2 = kMode == 1 ? 1 : 0;
  if (sdb_set_smem((const void*)nw_kernel<M2>, smem) != cudaSuccess)
    return SDB_ERR_CUDA;
  nw_kernel<M2><<<(unsigned)B, 32 * NW, smem, s>>>(theta, n, m, ws.wsb, ws.wsk, logz, marg, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

bool nw_fast_ok(int n, int m) {
  const int NW = (m + 1 + 31) / 32;
  return NW <= 32 && nw_smem_bytes(NW) <= 220 * 1024;
}

}  // namespace

// nw_gen.cu: anti-diagonal fp64 kernels for m beyond the strip kernels
bool nw_gen_ok(int n, int m);
size_t nw_gen_workspace(int64_t B, int n, int m, int mode);
int nw_gen_launch(int mode, const float* theta, int64_t B, int n, int m, void* ws, size_t ws_bytes, double* out,
                  float* marg, int8_t* path, int32_t* status, cudaStream_t s);

namespace {
int nw_check(int64_t B, int n, int m) {
  if (B < 0 || n < 1 || m < 1) return SDB_ERR_ARG;
  if (!nw_fast_ok(n, m) && !nw_gen_ok(n, m)) return SDB_ERR_UNSUPPORTED;
  return SDB_OK;
}
}  // namespace

extern "C" size_t sdb_nw_fb_workspace(int64_t B, int32_t n, int32_t m) {
  if (!nw_fast_ok(n, m)) return nw_gen_workspace(B, n, m, 1);
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
  if (!nw_fast_ok(n, m))
    return nw_gen_launch(marg ? 1 : 0, theta, B, n, m, workspace, ws_bytes, logz, marg, nullptr, status,
                         (cudaStream_t)stream);
  if (!marg) return nw_launch<0>(theta, B, n, m, NwWs{}, logz, nullptr, nullptr, nullptr, status, (cudaStream_t)stream);
  size_t need = 0;
  NwWs ws = nw_carve_ws(workspace, B, n, m, 1, &need);
  if (!workspace || ws_bytes < need) return SDB_ERR_WORKSPACE;
  return nw_launch<1>(theta, B, n, m, ws, logz, marg, nullptr, nullptr, status, (cudaStream_t)stream);
}

extern "C" size_t sdb_nw_viterbi_workspace(int64_t B, int32_t n, int32_t m) {
  if (!nw_fast_ok(n, m)) return nw_gen_workspace(B, n, m, 2);
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
  cudaStream_t s = (cudaStream_t)stream;
  if (!nw_fast_ok(n, m)) {
    if (sdb_note(cudaMemsetAsync(path, 0xff, (size_t)B * (n + 1) * (m + 1), s)) != cudaSuccess) return SDB_ERR_CUDA;
    return nw_gen_launch(2, theta, B, n, m, workspace, ws_bytes, score, nullptr, path, status, s);
  }
  size_t need = 0;
  NwWs ws = nw_carve_ws(workspace, B, n, m, 2, &need);
  if (!workspace || ws_bytes < need) return SDB_ERR_WORKSPACE;
  if (cudaMemsetAsync(path, 0xff, (size_t)B * (n + 1) * (m + 1), s) != cudaSuccess) return SDB_ERR_CUDA;
  return nw_launch<2>(theta, B, n, m, ws, nullptr, nullptr, path, score, status, s);
}
