// Projective spanning trees: Eisner inside/outside (log-partition, arc
// marginals) and the Kuhlmann arc-hybrid max-plus argmax.
//
// Reference: structdist spanning.py:183-280 (_eisner_charts,
// _eisner_root_terms, eisner_log_partition, eisner_marginals) and
// spanning.py:339-402 (_reweight_root, kuhlmann_argmax -- the public
// projective argmax).  Layout per instance: adjacency [n+1][n+1] fp32
// (head, dependent), position 0 = root.
//
// eisner_kernel -- one CTA (512 threads) per instance, n <= 128:
//   * the four inside charts cr, cl, ir, il and the three outside charts
//     ocr, ocl, ofold (ofold = outside of the shared split term; oir/oil are
//     consumed on the fly for the marginals) are packed upper-triangular fp32
//     arrays in shared memory (7 x n(n+1)/2 floats = 226 KB at n = 128);
//   * every value is stored relative to an INTEGER per-width offset
//     (Cin[w] for inside, Cout[w] for outside; a span of width w carries w
//     arcs, so offsets are re-chosen adaptively per width from the width's
//     max).  Integer offsets make every cross-width correction exact in fp32,
//     so all stored magnitudes stay small and fp32 keeps ~1e-6 absolute
//     accuracy at n = 128 (plain fp32 log-space would lose ~1e-4);
//   * inside by width (spanning.py:199-206), one warp per cell, lanes over
//     split points; outside by decreasing width in PULL form (each child
//     gathers from its parents, no atomics), marginals emitted per cell as
//     exp(o + i - Z) and clipped to [0,1] (spanning.py:280).
// kuhlmann_kernel -- fp64 max-plus tabulation over n+2 positions with the
// reference's scan order and strict '>' (first maximum), root reweighting for
// single-root, backtrack to heads[]; bit-exact with the reference.
#include "common.cuh"

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxN = 128;
static_assert(kMaxN <= 8 * kWarps, "per-width arc-weight prefetch: <= 8 spans per warp (16 lanes)");
constexpr int kQ = (kMaxN + 1 + 31) / 32;  // max split terms per lane

// packed strict-upper index over positions 0..n (i < j)
__device__ __forceinline__ int pk(int i, int j, int n) { return i * n - (i * (i - 1)) / 2 + (j - i - 1); }

size_t eisner_smem(int n) {
  const size_t T = (size_t)n * (n + 1) / 2;
  return 7 * T * 4 + (size_t)2 * (n + 2) * 4 + kWarps * 8 + 64;
}

struct Charts {
  float *cr, *cl, *ir, *il, *ocr, *ocl, *ofo;
  float *cin, *cout;
  float* wmax;
};

// complete charts: width-0 entries are 0 (cr[i,i] = cl[i,i] = 0)
__device__ __forceinline__ float cget(const float* c, int a, int b, int n) { return a == b ? 0.f : c[pk(a, b, n)]; }

// log-sum-exp of up to kQ per-lane terms, then across the warp
__device__ __forceinline__ float warp_lse_terms(const float (&t)[kQ]) {
  float m = ninf();
#pragma unroll
  for (int q = 0; q < kQ; ++q) m = fmaxf(m, t[q]);
  m = warp_max(m);
  float s = 0.f;
  if (m != ninf()) {
#pragma unroll
    for (int q = 0; q < kQ; ++q) s += ex2(t[q] - m);  // terms are in log2 units
  }
  s = warp_sum(s);
  return m == ninf() ? ninf() : m + lg2(s);
}

// All log values inside the kernel are in log2 units (x * log2 e): exp/log
// become single MUFU ops.  Integer offsets are integers in log2 units.
__global__ void __launch_bounds__(kThreads, 1) eisner_kernel(const float* __restrict__ adj_all, int n, int single,
                                                             double* __restrict__ logz, float* __restrict__ marg_all,
                                                             int32_t* __restrict__ status, int only_retry) {
  extern __shared__ __align__(16) char smraw[];
  if (only_retry && status[blockIdx.x] != 5) return;  // 5 = exp-space kernel gave up (kRetry)
  const int T = n * (n + 1) / 2;
  Charts c;
  {
    float* p = (float*)smraw;
    c.cr = p; p += T; c.cl = p; p += T; c.ir = p; p += T; c.il = p; p += T;
    c.ocr = p; p += T; c.ocl = p; p += T; c.ofo = p; p += T;
    c.cin = p; p += n + 2; c.cout = p; p += n + 2;
    c.wmax = p;
  }
  __shared__ int badsh;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N1 = n + 1;
  const float* th = adj_all + (size_t)b * N1 * N1;
  auto TH = [&](int h, int d) { return __ldg(th + h * N1 + d) * SDB_LOG2E; };
  if (tid == 0) badsh = 0;
  {
    int bad = 0;
    for (int e = tid; e < N1 * N1; e += kThreads) bad |= bad_input(th[e]);
    if (bad) atomicOr(&badsh, 1);
  }
  if (tid == 0) c.cin[0] = 0.f;
  __syncthreads();

  // ================================================================ inside
  for (int w = 1; w <= n; ++w) {
    const float Pw = (w == 1) ? 0.f : (w == 2 ? c.cin[1] : 2.f * c.cin[w - 1] - c.cin[w - 2]);
    if (tid == 0) c.cin[w] = Pw;
    __syncthreads();
    float lmax = ninf();
    for (int i = warp; i + w <= n; i += kWarps) {
      const int j = i + w;
      // fold = lse_{k in [i,j)} cr[i,k] + cl[k+1,j]   (widths k-i, j-k-1; sum w-1)
      float t[kQ];
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const int k = i + lane + 32 * q;
        t[q] = ninf();
        if (k < j) {
          const float x = cget(c.cr, i, k, n) + cget(c.cl, k + 1, j, n);
          t[q] = x + (c.cin[k - i] + c.cin[j - k - 1] - Pw);
        }
      }
      const float fold = warp_lse_terms(t);
      const float vir = (fold == ninf()) ? ninf() : TH(i, j) + fold;
      const float vil = (fold == ninf()) ? ninf() : TH(j, i) + fold;
      if (lane == 0) {
        c.ir[pk(i, j, n)] = vir;
        c.il[pk(i, j, n)] = vil;
      }
      __syncwarp();
      // cr = lse_{k in (i,j]} ir[i,k] + cr[k,j]; cl = lse_{k in [i,j)} cl[i,k] + il[k,j]
      float tr[kQ], tl[kQ];
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const int k = i + 1 + lane + 32 * q;  // (i, j]
        tr[q] = ninf();
        if (k <= j) tr[q] = c.ir[pk(i, k, n)] + cget(c.cr, k, j, n) + (c.cin[k - i] + c.cin[j - k] - Pw);
        const int k2 = i + lane + 32 * q;  // [i, j)
        tl[q] = ninf();
        if (k2 < j) tl[q] = cget(c.cl, i, k2, n) + c.il[pk(k2, j, n)] + (c.cin[k2 - i] + c.cin[j - k2] - Pw);
      }
      const float vcr = warp_lse_terms(tr);
      const float vcl = warp_lse_terms(tl);
      if (lane == 0) {
        c.cr[pk(i, j, n)] = vcr;
        c.cl[pk(i, j, n)] = vcl;
      }
      lmax = fmaxf(lmax, fmaxf(fmaxf(vir, vil), fmaxf(vcr, vcl)));
    }
    if (lane == 0) c.wmax[warp] = lmax;
    __syncthreads();
    float M = ninf();
#pragma unroll
    for (int q = 0; q < kWarps; ++q) M = fmaxf(M, c.wmax[q]);
    const float r = (M == ninf()) ? 0.f : rintf(M);
    if (r != 0.f) {
      for (int i = tid; i + w <= n; i += kThreads) {
        const int e = pk(i, i + w, n);
        c.ir[e] -= r; c.il[e] -= r; c.cr[e] -= r; c.cl[e] -= r;
      }
    }
    __syncthreads();
    if (tid == 0) c.cin[w] = Pw + r;
    __syncthreads();
  }

  // log Z (log2 units): value + integer offset
  __shared__ float zv, zc;  // Z = (zv + zc) log2 units
  if (tid == 0) {
    if (!single) {
      zv = c.cr[pk(0, n, n)];
      zc = c.cin[n];
    } else {
      // spanning.py:210-212: Z = lse_c th[0,c] + cl[1,c] + cr[c,n]
      float K = ninf();
      for (int cc = 1; cc <= n; ++cc) K = fmaxf(K, c.cin[cc - 1] + c.cin[n - cc]);
      float m = ninf();
      for (int cc = 1; cc <= n; ++cc) {
        const float x = TH(0, cc) + cget(c.cl, 1, cc, n) + cget(c.cr, cc, n, n) + (c.cin[cc - 1] + c.cin[n - cc] - K);
        m = fmaxf(m, x);
      }
      float s = 0.f;
      if (m != ninf())
        for (int cc = 1; cc <= n; ++cc) {
          const float x = TH(0, cc) + cget(c.cl, 1, cc, n) + cget(c.cr, cc, n, n) + (c.cin[cc - 1] + c.cin[n - cc] - K);
          s += ex2(x - m);
        }
      zv = (m == ninf()) ? ninf() : m + lg2(s);
      zc = K;
    }
  }
  __syncthreads();
  const bool zok = zv != ninf();
  if (tid == 0) {
    status[b] = badsh ? SDB_ST_INVALID : (zok ? SDB_ST_OK : SDB_ST_VACUOUS);
    logz[b] = zok ? ((double)zv + (double)zc) * (double)SDB_LN2 : ninfd();
  }
  if (!marg_all) return;
  float* mg = marg_all + (size_t)b * N1 * N1;
  if (!zok || badsh) {
    for (int e = tid; e < N1 * N1; e += kThreads) mg[e] = 0.f;
    return;
  }
  for (int e = tid; e < N1; e += kThreads) mg[e * N1 + e] = 0.f;
  if (single) {  // marg[0,c] = exp(root term - Z)
    for (int cc = 1 + tid; cc <= n; cc += kThreads) {
      const float x = TH(0, cc) + cget(c.cl, 1, cc, n) + cget(c.cr, cc, n, n) + (c.cin[cc - 1] + c.cin[n - cc] - zc);
      mg[cc] = fminf(fmaxf(ex2(x - zv), 0.f), 1.f);
    }
  }

  // =============================================================== outside
  // Pull form.  Offsets cout[w]; provisional Qw extrapolated from wider widths.
  for (int w = n; w >= 1; --w) {
    const float Qw = (w == n) ? 0.f : (w == n - 1 ? c.cout[n] : 2.f * c.cout[w + 1] - c.cout[w + 2]);
    if (tid == 0) c.cout[w] = Qw;
    __syncthreads();
    float lmax = ninf();
    for (int a = warp; a + w <= n; a += kWarps) {
      const int bb = a + w;
      // ---- ocr[a,bb]
      float tA[kQ], tB[kQ];
      // parents via the split term: j in (bb, n]: ofold[a,j] + cl[bb+1,j]
      // parents via cr: i in [0,a): ocr[i,bb] + ir[i,a]
      const int n1 = n - bb, n2 = a;
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const int x = lane + 32 * q;
        float tv = ninf();
        if (x < n1) {
          const int j = bb + 1 + x;
          tv = c.ofo[pk(a, j, n)] + cget(c.cl, bb + 1, j, n) + (c.cout[j - a] + c.cin[j - bb - 1] - Qw);
        } else if (x < n1 + n2) {
          const int i = x - n1;
          tv = c.ocr[pk(i, bb, n)] + c.ir[pk(i, a, n)] + (c.cout[bb - i] + c.cin[a - i] - Qw);
        }
        tA[q] = tv;
      }
      float vocr = warp_lse_terms(tA);
      // ---- ocl[a,bb]
      // split-term parents: i in [0, a-1]: ofold[i,bb] + cr[i,a-1]
      // cl parents: j in (bb, n]: ocl[a,j] + il[bb,j]
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const int x = lane + 32 * q;
        float tv = ninf();
        if (x < n2) {
          const int i = x;
          tv = c.ofo[pk(i, bb, n)] + cget(c.cr, i, a - 1, n) + (c.cout[bb - i] + c.cin[a - 1 - i] - Qw);
        } else if (x < n2 + n1) {
          const int j = bb + 1 + (x - n2);
          tv = c.ocl[pk(a, j, n)] + c.il[pk(bb, j, n)] + (c.cout[j - a] + c.cin[j - bb] - Qw);
        }
        tB[q] = tv;
      }
      float vocl = warp_lse_terms(tB);
      if (lane == 0) {
        // root seeds (spanning.py:233-245)
        if (!single) {
          if (a == 0 && bb == n) vocr = -Qw;  // ocr[0,n] = log 1 (multi-root Z = cr[0,n])
        } else {
          if (bb == n && a >= 1) {  // d root-term / d cr[a,n] = th[0,a] + cl[1,a]
            const float s0 = TH(0, a) + cget(c.cl, 1, a, n) + (c.cin[a - 1] - Qw);
            const float m = fmaxf(vocr, s0);
            if (m != ninf()) vocr = m + lg2(ex2(vocr - m) + ex2(s0 - m));
          }
          if (a == 1) {  // d root-term / d cl[1,bb] = th[0,bb] + cr[bb,n]
            const float s0 = TH(0, bb) + cget(c.cr, bb, n, n) + (c.cin[n - bb] - Qw);
            const float m = fmaxf(vocl, s0);
            if (m != ninf()) vocl = m + lg2(ex2(vocl - m) + ex2(s0 - m));
          }
        }
        c.ocr[pk(a, bb, n)] = vocr;
        c.ocl[pk(a, bb, n)] = vocl;
      }
      __syncwarp();
      // ---- oir[a,bb] = lse_{j in [bb,n]} ocr[a,j] + cr[bb,j]
      // ---- oil[a,bb] = lse_{i in [0,a]} ocl[i,bb] + cl[i,a]
      float tr[kQ], tl[kQ];
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const int x = lane + 32 * q;
        tr[q] = ninf();
        tl[q] = ninf();
        const int j = bb + x;
        if (j <= n) tr[q] = c.ocr[pk(a, j, n)] + cget(c.cr, bb, j, n) + (c.cout[j - a] + c.cin[j - bb] - Qw);
        if (x <= a) tl[q] = c.ocl[pk(x, bb, n)] + cget(c.cl, x, a, n) + (c.cout[bb - x] + c.cin[a - x] - Qw);
      }
      const float voir = warp_lse_terms(tr);
      const float voil = warp_lse_terms(tl);
      if (lane == 0) {
        const int e = pk(a, bb, n);
        const float thab = TH(a, bb), thba = TH(bb, a);
        // ofold = (oil + th[bb,a]) (+) (oir + th[a,bb])
        const float x1 = voil + thba, x2 = voir + thab;
        const float m = fmaxf(x1, x2);
        const float vof = (m == ninf()) ? ninf() : m + lg2(ex2(x1 - m) + ex2(x2 - m));
        c.ofo[e] = vof;
        // marginals: arc a->bb via ir, arc bb->a via il (spanning.py:264-277)
        const float off = (Qw + c.cin[w] - zc);
        const float pr = (voir == ninf() || c.ir[e] == ninf()) ? 0.f : ex2(voir + c.ir[e] + off - zv);
        const float pl = (voil == ninf() || c.il[e] == ninf()) ? 0.f : ex2(voil + c.il[e] + off - zv);
        if (!(single && a == 0)) mg[a * N1 + bb] = fminf(fmaxf(pr, 0.f), 1.f);
        mg[bb * N1 + a] = fminf(fmaxf(pl, 0.f), 1.f);
        lmax = fmaxf(lmax, fmaxf(fmaxf(vocr, vocl), vof));
      }
    }
    lmax = warp_max(lmax);
    if (lane == 0) c.wmax[warp] = lmax;
    __syncthreads();
    float M = ninf();
#pragma unroll
    for (int q = 0; q < kWarps; ++q) M = fmaxf(M, c.wmax[q]);
    const float r = (M == ninf()) ? 0.f : rintf(M);
    if (r != 0.f) {
      for (int a = tid; a + w <= n; a += kThreads) {
        const int e = pk(a, a + w, n);
        c.ocr[e] -= r; c.ocl[e] -= r; c.ofo[e] -= r;
      }
    }
    __syncthreads();
    if (tid == 0) c.cout[w] = Qw + r;
    __syncthreads();
  }
}

// ------------------------------------------------------------ exp space
// eisner_lin_kernel -- the same inside / pull-form outside in LINEAR space:
// every chart entry of width w is stored as exp(X) * 2^(-c w) for one slope
// c per instance (a tree has exactly n arcs, so scaling every arc weight by
// 2^-c scales each width-w product uniformly: W[h][d] = 2^(theta log2 e - c)).
// Every split term is then one FFMA (the log-space kernel needs ~20
// instructions: two-pass max / exp2 / offsets).  The slope adapts: when a
// width's largest entry leaves [2^-24, 2^24], c absorbs its per-width growth
// and all stored widths are rescaled by 2^(-delta width) (exact bookkeeping).
// Instances whose values overflow or underflow anyway (huge |theta| ranges,
// adversarial -inf patterns) report status 5 and are recomputed by the
// log-space eisner_kernel.  Adjoints G are pre-divided by E_Z, so an arc
// marginal is G_ir * E_ir.
constexpr int32_t kRetry = 5;

__device__ __forceinline__ float warp_dot_sum(float s) { return warp_sum(s); }
// Two warp sums in 5 shuffles (instead of 10): the xor-16 level exchanges the value the
// partner half keeps.  Lanes 0-15 end with sum(a), lanes 16-31 with sum(b).
__device__ __forceinline__ float warp_sum2(float a, float b, int lane) {
  const bool hi = lane & 16;
  float k = (hi ? b : a) + __shfl_xor_sync(0xffffffffu, hi ? a : b, 16);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
  return k;
}
// Four warp sums in 6 shuffles: lanes 0-7 end with sum(a), 8-15 sum(b), 16-23 sum(c),
// 24-31 sum(d).
__device__ __forceinline__ float warp_sum4(float a, float b, float c, float d, int lane) {
  const bool h16 = lane & 16, h8 = lane & 8;
  const float k0 = (h16 ? c : a) + __shfl_xor_sync(0xffffffffu, h16 ? a : c, 16);
  const float k1 = (h16 ? d : b) + __shfl_xor_sync(0xffffffffu, h16 ? b : d, 16);
  float k = (h8 ? k1 : k0) + __shfl_xor_sync(0xffffffffu, h8 ? k0 : k1, 8);
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
  return k;
}
// packed-row offset: chart[pk(x, c, n)] == chart[prow(x, n) + c]
__device__ __forceinline__ int prow(int x, int n) { return x * n - ((x * (x - 1)) >> 1) - x - 1; }

// 24 warps: 1.74 ms at C4 vs 1.82 (16 warps, 103 registers) and 1.86 (32 warps, 64 registers)
constexpr int kLinT = 768;
template <int kLT>
__global__ void __launch_bounds__(kLT, 1) eisner_lin_kernel(const float* __restrict__ adj_all, int n, int single,
                                                                 double* __restrict__ logz, float* __restrict__ marg_all,
                                                                 int32_t* __restrict__ status) {
  constexpr int kLW = kLT / 32;
  extern __shared__ __align__(16) char smraw[];
  const int T = n * (n + 1) / 2;
  float *cr, *cl, *ir, *il, *gcr, *gcl, *gfo;
  {
    float* p = (float*)smraw;
    cr = p; p += T; cl = p; p += T; ir = p; p += T; il = p; p += T;
    gcr = p; p += T; gcl = p; p += T; gfo = p; p += T;
  }
  __shared__ float wred[kLW], wred2[kLW];
  __shared__ float cslope, zv;
  __shared__ int badsh, failsh;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N1 = n + 1;
  const float* th = adj_all + (size_t)b * N1 * N1;
  // chart accessors: width-0 complete spans are 1
  auto CR = [&](int a, int bb) { return a == bb ? 1.f : cr[pk(a, bb, n)]; };
  auto CL = [&](int a, int bb) { return a == bb ? 1.f : cl[pk(a, bb, n)]; };
  if (tid == 0) { badsh = 0; failsh = 0; }
  // slope: mean finite theta (log2 units) over the dependents' incoming arcs
  {
    int bad = 0;
    float sum = 0.f, cnt = 0.f;
    for (int e = tid; e < N1 * N1; e += kLT) {
      const float x = th[e];
      bad |= bad_input(x);
      const int d = e % N1;
      if (d >= 1 && x != ninf() && x == x) { sum += x * SDB_LOG2E; cnt += 1.f; }
    }
    if (bad) atomicOr(&badsh, 1);
    sum = warp_sum(sum);
    cnt = warp_sum(cnt);
    if (lane == 0) { wred[warp] = sum; wred2[warp] = cnt; }
    __syncthreads();
    if (tid == 0) {
      float S = 0.f, C = 0.f;
      for (int q = 0; q < kLW; ++q) { S += wred[q]; C += wred2[q]; }
      cslope = (C > 0.f) ? rintf(S / C) : 0.f;
    }
    __syncthreads();
  }
  if (badsh) {  // status INVALID, zero marginals (as eisner_kernel)
    if (tid == 0) { status[b] = SDB_ST_INVALID; logz[b] = ninfd(); }
    if (marg_all) for (int e = tid; e < N1 * N1; e += kLT) marg_all[(size_t)b * N1 * N1 + e] = 0.f;
    return;
  }
  auto W = [&](int h, int d) { return ex2(__ldg(th + h * N1 + d) * SDB_LOG2E - cslope); };

  // ================================================================ inside
  for (int w = 1; w <= n; ++w) {
    float lmax = 0.f;
    // the arc weights of ALL this warp's spans of the width (<= 8 spans for n <= 128):
    // lane 2q / 2q+1 loads the right / left arc of span warp + q kLW, so one L2
    // latency per width is exposed instead of one per span pair
    float wpre;
    {
      const int q = lane >> 1, i = warp + q * kLW;
      wpre = (i + w <= n) ? ((lane & 1) ? W(i + w, i) : W(i, i + w)) : 0.f;
    }
    if (w <= 64) {
      // narrow widths: G = 2^lg lanes per span (<= 4 split terms per lane), 32 / G spans of
      // this warp per pass, reductions over lg shuffle levels inside each lane group
      const int lg = w <= 4 ? 0 : w <= 8 ? 1 : w <= 16 ? 2 : w <= 32 ? 3 : 4;
      const int G = 1 << lg, r = lane & (G - 1), qg = lane >> lg;
      for (int q0 = 0; warp + q0 * kLW + w <= n; q0 += 32 >> lg) {
        const int q = q0 + qg, i = warp + q * kLW, j = i + w;
        const bool ok = j <= n;
        const int src = 2 * min(q, 15);
        const float wr = __shfl_sync(0xffffffffu, wpre, src), wl = __shfl_sync(0xffffffffu, wpre, src + 1);
        float sf = 0.f;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int k = i + r + G * t;
          if (ok && k < j) sf = fmaf(CR(i, k), CL(k + 1, j), sf);
        }
        for (int o = G >> 1; o > 0; o >>= 1) sf += __shfl_xor_sync(0xffffffffu, sf, o);
        const float vir = wr * sf, vil = wl * sf;
        if (ok && r == 0) {
          ir[pk(i, j, n)] = vir;
          il[pk(i, j, n)] = vil;
        }
        __syncwarp();
        float sr = 0.f, sl = 0.f;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int o = r + G * t;
          if (ok && o < w) {
            sr = fmaf(ir[pk(i, i + 1 + o, n)], CR(i + 1 + o, j), sr);
            sl = fmaf(CL(i, i + o), il[pk(i + o, j, n)], sl);
          }
        }
        for (int o = G >> 1; o > 0; o >>= 1) {
          sr += __shfl_xor_sync(0xffffffffu, sr, o);
          sl += __shfl_xor_sync(0xffffffffu, sl, o);
        }
        if (ok && r == 0) {
          cr[pk(i, j, n)] = sr;
          cl[pk(i, j, n)] = sl;
        }
        if (ok) lmax = fmaxf(lmax, fmaxf(fmaxf(vir, vil), fmaxf(sr, sl)));
      }
      lmax = warp_max(lmax);
    } else
    // two spans per warp iteration: their reductions are independent (ILP)
    for (int i0 = warp, it = 0; i0 + w <= n; i0 += 2 * kLW, ++it) {
      const int iA = i0, iB = i0 + kLW;
      const bool hasB = iB + w <= n;
      const float wrA = __shfl_sync(0xffffffffu, wpre, 4 * it), wlA = __shfl_sync(0xffffffffu, wpre, 4 * it + 1);
      const float wrB = __shfl_sync(0xffffffffu, wpre, 4 * it + 2), wlB = __shfl_sync(0xffffffffu, wpre, 4 * it + 3);
      const int qi = (w + 31) >> 5;  // split terms per lane actually present at this width
      float sA = 0.f, sB = 0.f;
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        if (q >= qi) break;  // warp-uniform: only the 32-term slices this width needs
        const int kA = iA + lane + 32 * q, kB = iB + lane + 32 * q;
        if (kA < iA + w) sA = fmaf(CR(iA, kA), CL(kA + 1, iA + w), sA);
        if (hasB && kB < iB + w) sB = fmaf(CR(iB, kB), CL(kB + 1, iB + w), sB);
      }
      // lanes 0-15 hold F(A), lanes 16-31 F(B); lane 0 / lane 16 store span A / B
      const float F = warp_sum2(sA, sB, lane);
      const bool hiB = lane & 16;
      const float vir = (hiB ? wrB : wrA) * F, vil = (hiB ? wlB : wlA) * F;
      if (lane == 0) { ir[pk(iA, iA + w, n)] = vir; il[pk(iA, iA + w, n)] = vil; }
      if (lane == 16 && hasB) { ir[pk(iB, iB + w, n)] = vir; il[pk(iB, iB + w, n)] = vil; }
      lmax = fmaxf(lmax, fmaxf(vir, vil));
      __syncwarp();
      float srA = 0.f, slA = 0.f, srB = 0.f, slB = 0.f;
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        if (q >= qi) break;  // warp-uniform: only the 32-term slices this width needs
        const int o = lane + 32 * q;
        if (o + 1 <= w) srA = fmaf(ir[pk(iA, iA + 1 + o, n)], CR(iA + 1 + o, iA + w), srA);
        if (o < w) slA = fmaf(CL(iA, iA + o), il[pk(iA + o, iA + w, n)], slA);
        if (hasB) {
          if (o + 1 <= w) srB = fmaf(ir[pk(iB, iB + 1 + o, n)], CR(iB + 1 + o, iB + w), srB);
          if (o < w) slB = fmaf(CL(iB, iB + o), il[pk(iB + o, iB + w, n)], slB);
        }
      }
      // lanes 0 / 8 / 16 / 24 hold cr(A) / cl(A) / cr(B) / cl(B)
      const float v4 = warp_sum4(srA, slA, srB, slB, lane);
      if (lane == 0) cr[pk(iA, iA + w, n)] = v4;
      if (lane == 8) cl[pk(iA, iA + w, n)] = v4;
      if (hasB && lane == 16) cr[pk(iB, iB + w, n)] = v4;
      if (hasB && lane == 24) cl[pk(iB, iB + w, n)] = v4;
      lmax = fmaxf(lmax, v4);
    }
    if (lane == 0) wred[warp] = lmax;
    __syncthreads();
    float M = 0.f;
#pragma unroll
    for (int q = 0; q < kLW; ++q) M = fmaxf(M, wred[q]);
    if (!(M <= 3.0e38f)) {  // inf / NaN: give up on linear space
      if (tid == 0) failsh = 1;
      break;
    }
    if (M > 0.f && (M > 16777216.f || M < 5.9604645e-8f)) {
      // absorb the growth: c += delta, every stored width v scaled by 2^(-delta v)
      const float delta = lg2(M) / (float)w;
      for (int e = tid; e < T; e += kLT) {
        // decode width of packed (i, j): row i holds j = i+1..n
        int i = 0, r = e;
        while (r >= n - i) { r -= n - i; ++i; }
        const float f = ex2(-delta * (float)(r + 1));
        cr[e] *= f; cl[e] *= f; ir[e] *= f; il[e] *= f;
      }
      __syncthreads();
      if (tid == 0) cslope += delta;
    }
    __syncthreads();
  }
  // Z (spanning.py:210-221)
  if (tid == 0 && !failsh) {
    float ez;
    if (!single) {
      ez = CR(0, n);
    } else {
      ez = 0.f;
      for (int cc = 1; cc <= n; ++cc) ez += W(0, cc) * CL(1, cc) * CR(cc, n);
    }
    zv = ez;
    // zero can be a true -inf (vacuous) or an underflow: let the log-space kernel decide
    if (!(ez > 0.f) || !(ez <= 3.0e38f)) failsh = 1;
  }
  __syncthreads();
  if (failsh) {
    if (tid == 0) status[b] = kRetry;
    return;
  }
  const float EZ = zv;
  if (tid == 0) {
    status[b] = SDB_ST_OK;
    logz[b] = ((double)lg2(EZ) + (double)cslope * (double)n) * (double)SDB_LN2;
  }
  if (!marg_all) return;
  float* mg = marg_all + (size_t)b * N1 * N1;
  const float rz = 1.f / EZ;
  for (int e = tid; e < N1; e += kLT) mg[e * N1 + e] = 0.f;
  if (single)
    for (int cc = 1 + tid; cc <= n; cc += kLT)
      mg[cc] = fminf(fmaxf(W(0, cc) * CL(1, cc) * CR(cc, n) * rz, 0.f), 1.f);

  // =============================================================== outside
  // column reads chart[pk(x, c)] for x = lane + 32 q: per-lane packed-row offsets
  int Rq[kQ];
#pragma unroll
  for (int q = 0; q < kQ; ++q) Rq[q] = prow(lane + 32 * q, n);
  for (int w = n; w >= 1; --w) {
    float lmax = 0.f;
    float wpre;  // this warp's arc weights of the width, as in the inside pass
    {
      const int q = lane >> 1, a = warp + q * kLW;
      wpre = (a + w <= n) ? ((lane & 1) ? W(a, a + w) : W(a + w, a)) : 0.f;
    }
    // two spans per warp iteration (A = a, B = a + kLW): independent chains in flight
    for (int a = warp, it = 0; a + w <= n; a += 2 * kLW, it += 2) {
      const bool hasB = a + kLW + w <= n;
      float sv[2][2], wv[2][2];
      int bq[2], rA[2], rB[2], rB1[2], n1q[2], n2q[2];
      int qo1 = 0, qo2 = 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int aa = a + h * kLW, bb = aa + w;
        const bool live = h == 0 || hasB;
        bq[h] = bb;
        n1q[h] = live ? n - bb : 0;
        n2q[h] = live ? aa : 0;
        rA[h] = prow(aa, n);
        rB[h] = prow(bb, n);
        rB1[h] = prow(bb + 1, n);
        wv[h][0] = __shfl_sync(0xffffffffu, wpre, 2 * (it + h));      // W(bb, aa)
        wv[h][1] = __shfl_sync(0xffffffffu, wpre, 2 * (it + h) + 1);  // W(aa, bb)
        sv[h][0] = sv[h][1] = 0.f;
        if (live) {
          qo1 = max(qo1, (max(n1q[h], n2q[h]) + 31) >> 5);
          qo2 = max(qo2, (max(n1q[h], aa) + 32) >> 5);
        }
      }
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        if (q >= qo1) break;  // warp-uniform: only the 32-term slices this width needs
        const int x = lane + 32 * q;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int aa = a + h * kLW, bb = bq[h];
          const bool pr = x < n1q[h], pl = x < n2q[h];
          const int j = bb + 1 + x;
          // right parents (aa, j): split (gfo) with CL(bb+1, j) (1 at j = bb+1), cl parents with il(bb, j)
          const float g1 = pr ? gfo[rA[h] + j] : 0.f, c1 = (pr && x > 0) ? cl[rB1[h] + j] : 1.f;
          const float g2 = pr ? gcl[rA[h] + j] : 0.f, c2 = pr ? il[rB[h] + j] : 0.f;
          // left parents (x, bb): cr parents with ir(x, aa), split (gfo) with CR(x, aa-1) (1 at x = aa-1)
          const float g3 = pl ? gcr[Rq[q] + bb] : 0.f, c3 = pl ? ir[Rq[q] + aa] : 0.f;
          const float g4 = pl ? gfo[Rq[q] + bb] : 0.f, c4 = (pl && x != aa - 1) ? cr[Rq[q] + aa - 1] : 1.f;
          sv[h][0] = fmaf(g1, c1, fmaf(g3, c3, sv[h][0]));
          sv[h][1] = fmaf(g2, c2, fmaf(g4, c4, sv[h][1]));
        }
      }
      // lanes 0 / 8 / 16 / 24: cr adjoint of A / cl adjoint of A / cr of B / cl of B
      {
        const float vg = warp_sum4(sv[0][0], sv[0][1], sv[1][0], sv[1][1], lane);
        const int h = lane >> 4, aa = a + h * kLW, bb = aa + w;
        if ((lane & 15) == 0 && (h == 0 || hasB)) {
          float v = vg;
          if (!single) {
            if (aa == 0 && bb == n) v = rz;
          } else {
            if (bb == n && aa >= 1) v += W(0, aa) * CL(1, aa) * rz;
          }
          gcr[pk(aa, bb, n)] = v;
          lmax = fmaxf(lmax, v);
        }
        if ((lane & 15) == 8 && (h == 0 || hasB)) {
          float v = vg;
          if (single && aa == 1) v += W(0, bb) * CR(bb, n) * rz;
          gcl[pk(aa, bb, n)] = v;
          lmax = fmaxf(lmax, v);
        }
      }
      __syncwarp();
      float tv[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        if (q >= qo2) break;  // warp-uniform: only the 32-term slices this width needs
        const int x = lane + 32 * q;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int aa = a + h * kLW, bb = bq[h];
          const bool live = h == 0 || hasB;
          const int j = bb + x;
          const bool pr = live && j <= n, pl = live && x <= aa;
          const float g1 = pr ? gcr[rA[h] + j] : 0.f, c1 = (pr && x > 0) ? cr[rB[h] + j] : 1.f;  // CR(bb, j)
          const float g2 = pl ? gcl[Rq[q] + bb] : 0.f, c2 = (pl && x != aa) ? cl[Rq[q] + aa] : 1.f;  // CL(x, aa)
          tv[h][0] = fmaf(g1, c1, tv[h][0]);
          tv[h][1] = fmaf(g2, c2, tv[h][1]);
        }
      }
      // lanes 0 / 8 / 16 / 24: ir adjoint of A / il of A / ir of B / il of B
      const float gt = warp_sum4(tv[0][0], tv[0][1], tv[1][0], tv[1][1], lane);
      const float gl8 = __shfl_down_sync(0xffffffffu, gt, 8);
      {
        const int h = lane >> 4, aa = a + h * kLW, bb = aa + w;
        if ((lane & 15) == 0 && (h == 0 || hasB)) {
          const int e = pk(aa, bb, n);
          const float gir = gt, gil = gl8;
          const float vf = gil * (h ? wv[1][0] : wv[0][0]) + gir * (h ? wv[1][1] : wv[0][1]);
          gfo[e] = vf;
          const float pr = gir * ir[e], pl = gil * il[e];
          if (!(single && aa == 0)) mg[aa * N1 + bb] = fminf(fmaxf(pr, 0.f), 1.f);
          mg[bb * N1 + aa] = fminf(fmaxf(pl, 0.f), 1.f);
          lmax = fmaxf(lmax, vf);
        }
      }
    }
    lmax = warp_max(lmax);
    if (lane == 0) wred[warp] = lmax;
    __syncthreads();
    float M = 0.f;
#pragma unroll
    for (int q = 0; q < kLW; ++q) M = fmaxf(M, wred[q]);
    if (!(M <= 3.0e38f)) {
      if (tid == 0) status[b] = kRetry;
      return;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- Kuhlmann
// fp64 max-plus over positions 0..n+1 (n+1 = end marker, heads nothing).
// table packed strict-upper over N2 = n+2 positions; back = (k, head).
size_t kuhl_smem(int n) {
  const size_t N2 = n + 2;
  const size_t T = N2 * (N2 - 1) / 2;
  return T * 8 + T * 4 + 64;
}

__device__ __forceinline__ int pk2(int i, int j, int N) { return i * (N - 1) - (i * (i - 1)) / 2 + (j - i - 1); }

// kGlobal: table and back pointers in global scratch (n beyond shared memory)
template <bool kGlobal>
__global__ void __launch_bounds__(kThreads, 2) kuhlmann_kernel(const float* __restrict__ adj_all, int n, int single,
                                                               int32_t* __restrict__ heads_all,
                                                               double* __restrict__ score,
                                                               int32_t* __restrict__ status, char* __restrict__ gscr) {
  extern __shared__ __align__(16) char smraw[];
  const int N = n + 2;
  const int T = N * (N - 1) / 2;
  double* tab = kGlobal ? (double*)(gscr + (size_t)blockIdx.x * (((size_t)T * 12 + 15) & ~(size_t)15))
                       : (double*)smraw;
  int* back = (int*)(tab + T);  // (k << 1) | (head == j)
  __shared__ double rw_c;
  __shared__ int badsh;
  __shared__ float fmax_s;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N1 = n + 1;
  const float* th = adj_all + (size_t)b * N1 * N1;
  if (tid == 0) { badsh = 0; fmax_s = ninf(); }
  __syncthreads();
  {
    int bad = 0;
    float lo = __int_as_float(0x7f800000), hi = ninf();
    for (int e = tid; e < N1 * N1; e += kThreads) {
      const float x = th[e];
      bad |= bad_input(x);
      if (x != ninf() && x == x && x != __int_as_float(0x7f800000)) { lo = fminf(lo, x); hi = fmaxf(hi, x); }
    }
    if (bad) atomicOr(&badsh, 1);
    lo = -warp_max(-lo);
    hi = warp_max(hi);
    __shared__ float lo_w[kWarps], hi_w[kWarps];
    if (lane == 0) { lo_w[warp] = lo; hi_w[warp] = hi; }
    __syncthreads();
    if (tid == 0) {
      float L = lo_w[0], H = hi_w[0];
      for (int q = 1; q < kWarps; ++q) { L = fminf(L, lo_w[q]); H = fmaxf(H, hi_w[q]); }
      fmax_s = H;
      // spanning.py:339-350: c = n * (max - min) + 1 over the finite entries
      rw_c = (double)n * ((double)H - (double)L) + 1.0;
    }
    __syncthreads();
  }
  const bool no_finite = (fmax_s == ninf());
  // score(h, k): reweighted th[h][k] for h in 0..n, k in 1..n; end marker heads nothing
  auto S = [&](int h, int k) -> double {
    if (h > n || k < 1 || k > n) return ninfd();
    double v = (double)__ldg(th + h * N1 + k);
    if (single && h == 0) v = v - rw_c;
    return v;
  };
  for (int e = tid; e < T; e += kThreads) tab[e] = ninfd();
  __syncthreads();
  for (int i = tid; i + 1 < N; i += kThreads) tab[pk2(i, i + 1, N)] = 0.0;
  __syncthreads();
  // G = 2^lg lanes per span (<= 4 split points per lane): narrow widths put
  // many spans in a warp instead of one span with mostly idle lanes
  for (int w = 2; w < N; ++w) {
    const int nsp = N - w, L = w - 1;
    const int x = (L - 1) >> 2;
    const int lg = min(5, x > 0 ? 32 - __clz(x) : 0), G = 1 << lg, r = lane & (G - 1);
    const int wfirst = (tid & ~31) >> lg;
    for (int base = 0; base < nsp; base += kThreads >> lg) {
      if (base + wfirst >= nsp) break;  // warp-uniform
      const int i0 = base + (tid >> lg);
      const bool ok = i0 < nsp;
      const int i = ok ? i0 : 0, j = i + w;
      // candidates in reference order: k ascending, head i then head j; strict '>'
      double best = ninfd();
      int arg = 0x7fffffff;  // encoded order index 2*(k-i-1) + (head==j)
      if (ok) {
        for (int k = i + 1 + r; k < j; k += G) {
          // arc scores first: the global (L2) loads overlap the shared-memory chart reads
          const double s1 = S(i, k), s2 = S(j, k);
          const double base2 = tab[pk2(i, k, N)] + tab[pk2(k, j, N)];
          if (base2 == ninfd()) continue;
          const double c1 = base2 + s1, c2 = base2 + s2;
          const int o = 2 * (k - i - 1);
          if (c1 > best) { best = c1; arg = o; }
          if (c2 > best) { best = c2; arg = o + 1; }
        }
      }
      for (int o = G >> 1; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
        if (ov > best || (ov == best && oa < arg)) { best = ov; arg = oa; }
      }
      if (ok && r == 0) {
        tab[pk2(i, j, N)] = best;
        back[pk2(i, j, N)] = (arg == 0x7fffffff) ? -1 : arg;
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    int32_t* heads = heads_all + (size_t)b * N1;
    const double top = tab[pk2(0, N - 1, N)];
    int st = (badsh) ? SDB_ST_INVALID : ((top == ninfd() || no_finite) ? SDB_ST_VACUOUS : SDB_ST_OK);
    for (int d = 0; d <= n; ++d) heads[d] = -1;
    if (st == SDB_ST_OK) {
      // explicit stack (reuse the tail of back[] is unsafe; use a small local stack in registers via shared)
      int* stk = (int*)(tab);  // table no longer needed except top; safe to reuse
      int sp = 0;
      stk[sp++] = 0;
      stk[sp++] = N - 1;
      int roots = 0;
      while (sp > 0) {
        const int j = stk[--sp];
        const int i = stk[--sp];
        if (j == i + 1) continue;
        const int code = back[pk2(i, j, N)];
        const int k = i + 1 + (code >> 1);
        const int h = (code & 1) ? j : i;
        heads[k] = h;
        if (h == 0) ++roots;
        stk[sp++] = i; stk[sp++] = k;
        stk[sp++] = k; stk[sp++] = j;
      }
      if (single && roots != 1) st = SDB_ST_VACUOUS;
      if (st != SDB_ST_OK)
        for (int d = 0; d <= n; ++d) heads[d] = -1;
    }
    status[b] = st;
    score[b] = top;
  }
}

bool eisner_fast_ok(int n) { return n <= kMaxN && eisner_smem(n) <= 227 * 1024; }

int eisner_check(int64_t B, int n) {
  if (B < 0 || n < 1) return SDB_ERR_ARG;
  if (n > 4096) return SDB_ERR_UNSUPPORTED;
  return SDB_OK;
}

}  // namespace

// eisner_gen.cu: fp64 charts in global memory for n > 128
int eisner_gen_launch(const float* adj, int64_t B, int n, int single, double* logz, float* marg, int32_t* status,
                      cudaStream_t s);

extern "C" int sdb_eisner(const float* adjacency, int64_t B, int32_t n, int32_t single_root, double* logz,
                          float* marg, int32_t* status, void* stream) {
  int rc = eisner_check(B, n);
  if (rc) return rc;
  if (!adjacency || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!eisner_fast_ok(n))
    return eisner_gen_launch(adjacency, B, n, single_root ? 1 : 0, logz, marg, status, (cudaStream_t)stream);
  const size_t smem = eisner_smem(n);
  const size_t smem_lin = (size_t)7 * (n * (n + 1) / 2) * 4;  // the seven charts only
  cudaStream_t s = (cudaStream_t)stream;
  if (sdb_set_smem((const void*)eisner_lin_kernel<kLinT>, smem_lin) != cudaSuccess ||
      sdb_set_smem((const void*)eisner_kernel, smem) != cudaSuccess)
    return SDB_ERR_CUDA;
  // exp-space first; the log-space kernel redoes only the instances it flagged
  eisner_lin_kernel<kLinT><<<(unsigned)B, kLinT, smem_lin, s>>>(adjacency, n, single_root ? 1 : 0, logz, marg, status);
  SDB_CHECK_LAUNCH();
  eisner_kernel<<<(unsigned)B, kThreads, smem, s>>>(adjacency, n, single_root ? 1 : 0, logz, marg, status, 1);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" int sdb_kuhlmann(const float* adjacency, int64_t B, int32_t n, int32_t single_root, int32_t* heads,
                            double* score, int32_t* status, void* stream) {
  if (B < 0 || n < 1) return SDB_ERR_ARG;
  if (n > 8192) return SDB_ERR_UNSUPPORTED;
  if (!adjacency || !heads || !score || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t smem = kuhl_smem(n);
  if (smem > 227 * 1024) {  // tables in stream-ordered global scratch (no workspace argument)
    const size_t N2 = n + 2, T = N2 * (N2 - 1) / 2;
    void* scr = nullptr;
    if (sdb_note(cudaMallocAsync(&scr, (size_t)B * ((T * 12 + 15) & ~(size_t)15), s)) != cudaSuccess)
      return SDB_ERR_CUDA;
    kuhlmann_kernel<true><<<(unsigned)B, kThreads, 0, s>>>(adjacency, n, single_root ? 1 : 0, heads, score, status,
                                                          (char*)scr);
    SDB_CHECK_LAUNCH();
    return sdb_note(cudaFreeAsync(scr, s)) == cudaSuccess ? SDB_OK : SDB_ERR_CUDA;
  }
  if (sdb_set_smem((const void*)kuhlmann_kernel<false>, smem) != cudaSuccess)
    return SDB_ERR_CUDA;
  kuhlmann_kernel<false><<<(unsigned)B, kThreads, smem, s>>>(adjacency, n, single_root ? 1 : 0, heads, score, status,
                                                             nullptr);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
