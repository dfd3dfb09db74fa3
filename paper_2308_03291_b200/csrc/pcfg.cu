// PCFG (Chomsky normal form): inside log-partition and constituent (span)
// marginals via inside/outside in scaled linear space; max-plus argmax.
//
// Reference: structdist constituency.py:246-371 (_pcfg_inside, pcfg_inside,
// pcfg_gradients, _pcfg_walk, pcfg_argmax).  Per instance: root [NT],
// binary_rules [NT][S][S] (children: NTs 0..NT-1 then PTs NT..S-1),
// emissions [n][PT], optional sticky [n][n] in {0,-inf}.  NT, PT <= 32,
// n <= 64.
//
// Representation: each chart cell (i,j) holds a fp64 log scale s_ij and a
// fp32 vector u_ij[32] = exp(chart[i,j,X] - s_ij) over its symbol class (PT
// for width-1 spans, NT for wider spans).  All products are then positive
// linear-space FMAs; logs/exps are O(spans).
//
// Inside, width w (all spans of the width together, one CTA per instance):
//   P-build: warp per span; P_t[B][C] = sum_k f_k u_ik[B] u_(k+1)j[C] with
//            f_k = exp(s_ik + s_(k+1)j - Smax), split into the <= 3 child-class
//            blocks t (leaf/NT x leaf/NT) -> global scratch;
//   contraction: inner[A] = sum_t sum_{B,C} R_t[A,B,C] P_t[B,C], a GEMM over
//            K = 3*32*32 with N = spans of the width, R (= exp rules) streamed
//            once per width through shared memory in B-slices; register-
//            blocked over the warp's spans (lane = A).
// Outside, parent width w descending (push form, constituency.py:303-325):
//   Q-build: Q_p[t][B][C] = sum_A o_p[A] R_t[A,B,C] (lane = C, register-blocked
//            over parents, R in B-slices through shared memory);
//   left pushes then right pushes (each child receives <= 1 push of each kind
//   per parent width, so no atomics), merged into the child's scaled vector.
// Span marginals: exp(o_s + i_s - Z) * sum_X o[X] u[X].
#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kSpW = 8;    // spans per warp (register block); n <= 64
constexpr int kBS = 4;     // B-slice width
constexpr int kMaxN = 64;

struct PcfgWs {
  float* RE;    // [B][4][32 A][32 B][32 C]  exp(rules) per child-class block t, zero padded
  float* RT;    // [B][4][32 B][32 C][32 A]  the same, A fastest (inside contraction)
  float* iu;    // [B][n][n][32]
  double* isc;  // [B][n][n]
  float* ou;    // [B][n][n][32]
  double* osc;  // [B][n][n]
  float* P;     // [B][n][3][32][32] per-width scratch (P in inside, Q in outside)
  float* Q2;    // [B][n][3][32][32] transposed Q for left pushes
};

PcfgWs pcfg_carve(void* base, int64_t B, int n, int NT, int PT, size_t* bytes) {
  const size_t S = NT + PT;
  Carve c(base);
  PcfgWs w;
  w.RE = c.take<float>((size_t)B * 4 * 32768);  // REp[t][A][B][C] zero-padded per child block
  w.RT = c.take<float>((size_t)B * 4 * 32768);  // RTp[t][B][C][A]
  w.iu = c.take<float>((size_t)B * n * n * 32);
  w.isc = c.take<double>((size_t)B * n * n);
  w.ou = c.take<float>((size_t)B * n * n * 32);
  w.osc = c.take<double>((size_t)B * n * n);
  w.P = c.take<float>((size_t)B * n * 3 * 1024);
  w.Q2 = c.take<float>((size_t)B * n * 3 * 1024);
  *bytes = c.used;
  return w;
}

__device__ __forceinline__ void cpa16(float* dst, const float* src) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
}
__device__ __forceinline__ void cpa_commit_wait() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
  __syncthreads();
}

// child class offsets of block t: t0 = (NT,NT) t1 = (PT,NT) t2 = (NT,PT) t3 = (PT,PT)
__device__ __forceinline__ int boff(int t, int NT) { return (t == 1 || t == 3) ? NT : 0; }
__device__ __forceinline__ int coff(int t, int NT) { return (t == 2 || t == 3) ? NT : 0; }
__device__ __forceinline__ int bcnt(int t, int NT, int PT) { return (t == 1 || t == 3) ? PT : NT; }
__device__ __forceinline__ int ccnt(int t, int NT, int PT) { return (t == 2 || t == 3) ? PT : NT; }
// block of slot `sl` at width w: w == 2 -> only slot 0 = t3; else slot 0 = t0 (interior), 1 = t1 (k=i), 2 = t2 (k=j-1)
__device__ __forceinline__ int slot_type(int sl, int w) { return w == 2 ? 3 : sl; }

template <bool kMarg>
__global__ void __launch_bounds__(kThreads, 1) pcfg_kernel(
    const float* __restrict__ root_all, const float* __restrict__ rules_all, const float* __restrict__ emis_all,
    const float* __restrict__ sticky_all, int n, int NT, int PT, PcfgWs ws, double* __restrict__ logz,
    float* __restrict__ marg_all, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) float smf[];
  const int S = NT + PT;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* root = root_all + (size_t)b * NT;
  const float* rules = rules_all + (size_t)b * NT * S * S;
  const float* emis = emis_all + (size_t)b * n * PT;
  const float* sticky = sticky_all ? sticky_all + (size_t)b * n * n : nullptr;
  float* RE = ws.RE + (size_t)b * 4 * 32768;
  float* RT = ws.RT + (size_t)b * 4 * 32768;
  float* iu = ws.iu + (size_t)b * n * n * 32;
  double* isc = ws.isc + (size_t)b * n * n;
  float* ou = ws.ou + (size_t)b * n * n * 32;
  double* osc = ws.osc + (size_t)b * n * n;
  float* Pw = ws.P + (size_t)b * n * 3 * 1024;
  float* Q2 = ws.Q2 + (size_t)b * n * 3 * 1024;
  __shared__ int badsh;
  __shared__ double smax_s[kMaxN];
  if (tid == 0) badsh = 0;
  __syncthreads();
  auto STK = [&](int i, int j) -> float { return sticky ? sticky[i * n + j] : 0.f; };

  // ---- prologue: exp(rules) into zero-padded per-block layouts (RE: C fastest, RT: A fastest),
  // input checks
  {
    int bad = 0;
    for (int e = tid; e < NT * S * S; e += kThreads) bad |= bad_input(rules[e]);
    for (int e = tid; e < 4 * 32768; e += kThreads) {
      const int t = e >> 15, r = e & 32767;
      const int A = r >> 10, Bi = (r >> 5) & 31, C = r & 31;
      float v = 0.f;
      if (A < NT && Bi < bcnt(t, NT, PT) && C < ccnt(t, NT, PT))
        v = fexp(rules[((size_t)A * S + boff(t, NT) + Bi) * S + coff(t, NT) + C]);
      RE[e] = v;                                              // [t][A][B][C]
      RT[(((size_t)t * 32 + Bi) * 32 + C) * 32 + A] = v;      // [t][B][C][A]
    }
    for (int e = tid; e < NT; e += kThreads) bad |= bad_input(root[e]);
    for (int e = tid; e < n * PT; e += kThreads) bad |= bad_input(emis[e]);
    if (sticky)
      for (int e = tid; e < n * n; e += kThreads) bad |= !(sticky[e] == 0.f || sticky[e] == ninf());
    if (bad) atomicOr(&badsh, 1);
  }
  __syncthreads();
  // ---- width 1: preterminal slots (constituency.py:257-258)
  for (int i = warp; i < n; i += kWarps) {
    const float x = (lane < PT) ? emis[i * PT + lane] : ninf();
    const float m = warp_max(x);
    const float st = STK(i, i);
    const bool dead = (m == ninf()) || st == ninf();
    iu[(size_t)(i * n + i) * 32 + lane] = dead ? 0.f : fexp(x - m);
    if (lane == 0) isc[i * n + i] = dead ? ninfd() : (double)m;
  }
  __syncthreads();

  float* RTs = smf;                 // [3][kBS][32 C][32 A]
  float* Ps = smf + 3 * kBS * 1024; // [kMaxN spans][3][kBS][32 C]

  // ================================================================ inside
  for (int w = 2; w <= n; ++w) {
    const int nsp = n - w + 1;
    const int nslot = (w == 2) ? 1 : 3;
    // ---- P-build: warp per span
    for (int i = warp; i < nsp; i += kWarps) {
      const int j = i + w - 1;
      double sm = ninfd();
      for (int k = i + lane; k < j; k += 32) sm = fmax(sm, isc[i * n + k] + isc[(k + 1) * n + j]);
      sm = warp_maxd(sm);
      if (lane == 0) smax_s[i] = sm;
      float acc[3][32];
#pragma unroll
      for (int sl = 0; sl < 3; ++sl)
#pragma unroll
        for (int q = 0; q < 32; ++q) acc[sl][q] = 0.f;
      if (sm != ninfd()) {
        for (int k = i; k < j; ++k) {
          const double sk = isc[i * n + k] + isc[(k + 1) * n + j];
          if (sk == ninfd()) continue;
          const float f = fexp((float)(sk - sm));
          const float lv = iu[(size_t)(i * n + k) * 32 + lane];
          const float rv = iu[(size_t)((k + 1) * n + j) * 32 + lane] * f;  // lane = C
          const int sl = (w == 2) ? 0 : (k == i ? 1 : (k == j - 1 ? 2 : 0));
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const float lb = __shfl_sync(0xffffffffu, lv, q);
            if (sl == 0) acc[0][q] = fmaf(lb, rv, acc[0][q]);
            else if (sl == 1) acc[1][q] = fmaf(lb, rv, acc[1][q]);
            else acc[2][q] = fmaf(lb, rv, acc[2][q]);
          }
        }
      }
      float* pp = Pw + (size_t)i * 3 * 1024;
#pragma unroll
      for (int sl = 0; sl < 3; ++sl)
#pragma unroll
        for (int q = 0; q < 32; ++q) pp[sl * 1024 + q * 32 + lane] = acc[sl][q];  // [slot][B][C]
    }
    __syncthreads();
    // ---- contraction: inner[s][A] = sum_{slot,B,C} R_t[A,B',C'] P[s][slot][B][C]
    float inner[kSpW];
#pragma unroll
    for (int q = 0; q < kSpW; ++q) inner[q] = 0.f;
    for (int b0 = 0; b0 < 32; b0 += kBS) {
      // stage R slice RTs[sl][bb][C][A] (4 KB contiguous per (sl, bb)) and the P slice
      // Ps[s][sl][bb][C] (512 B contiguous per (s, sl)) with 16-byte cp.async
      for (int e = tid; e < nslot * kBS * 256; e += kThreads) {
        const int sl = e / (kBS * 256), r = e - sl * (kBS * 256);
        const int t = slot_type(sl, w);
        cpa16(RTs + sl * kBS * 1024 + 4 * r, RT + ((size_t)t * 32 + b0) * 1024 + 4 * r);
      }
      for (int e = tid; e < nsp * nslot * 32; e += kThreads) {
        const int s2 = e / (nslot * 32), r = e - s2 * (nslot * 32);
        const int sl = r >> 5, q = r & 31;
        cpa16(Ps + (s2 * 3 + sl) * kBS * 32 + 4 * q, Pw + (size_t)s2 * 3 * 1024 + sl * 1024 + b0 * 32 + 4 * q);
      }
      cpa_commit_wait();
      __syncthreads();
      for (int sl = 0; sl < nslot; ++sl) {
        for (int bb = 0; bb < kBS; ++bb) {
#pragma unroll 4
          for (int C = 0; C < 32; C += 4) {
            const float r0 = RTs[((sl * kBS + bb) * 32 + C + 0) * 32 + lane];
            const float r1 = RTs[((sl * kBS + bb) * 32 + C + 1) * 32 + lane];
            const float r2 = RTs[((sl * kBS + bb) * 32 + C + 2) * 32 + lane];
            const float r3 = RTs[((sl * kBS + bb) * 32 + C + 3) * 32 + lane];
#pragma unroll
            for (int q = 0; q < kSpW; ++q) {
              const int s = warp + q * kWarps;
              if (s < nsp) {
                const float4 p = *reinterpret_cast<const float4*>(&Ps[((s * 3 + sl) * kBS + bb) * 32 + C]);
                inner[q] = fmaf(r0, p.x, fmaf(r1, p.y, fmaf(r2, p.z, fmaf(r3, p.w, inner[q]))));
              }
            }
          }
        }
      }
      __syncthreads();
    }
    // ---- normalise and store the width's cells (constituency.py:264-265)
#pragma unroll
    for (int q = 0; q < kSpW; ++q) {
      const int i = warp + q * kWarps;
      if (i < nsp) {
        const int j = i + w - 1;
        const float v = (lane < NT) ? inner[q] : 0.f;
        const float m = warp_max(v);
        const double sm = smax_s[i];
        const float st = STK(i, j);
        const bool dead = !(m > 0.f) || sm == ninfd() || st == ninf();
        iu[(size_t)(i * n + j) * 32 + lane] = dead ? 0.f : v / m;
        if (lane == 0) isc[i * n + j] = dead ? ninfd() : sm + (double)flog(m);
      }
    }
    __syncthreads();
  }

  // log Z = lse_A root[A] + chart[0,n-1,A] (constituency.py:271)
  __shared__ double zsh;
  if (warp == 0) {
    const double s0 = isc[n - 1];
    const float r = (lane < NT) ? root[lane] : ninf();
    const float rm = warp_max(r);
    const float v = (lane < NT && rm != ninf()) ? fexp(r - rm) * iu[(size_t)(n - 1) * 32 + lane] : 0.f;
    const float tot = warp_sum(v);
    // a width-1 root span holds only preterminals: no derivation (constituency.py:271)
    if (lane == 0) zsh = (n == 1 || s0 == ninfd() || !(tot > 0.f)) ? ninfd() : s0 + (double)rm + (double)flog(tot);
  }
  __syncthreads();
  const double Z = zsh;
  if (tid == 0) {
    status[b] = badsh ? SDB_ST_INVALID : (Z == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
    logz[b] = Z;
  }
  if (!kMarg) return;
  float* mg = marg_all + (size_t)b * n * n;
  if (Z == ninfd() || badsh) {
    for (int e = tid; e < n * n; e += kThreads) mg[e] = 0.f;
    return;
  }

  // =============================================================== outside
  for (int e = tid; e < n * n; e += kThreads) osc[e] = ninfd();
  for (int e = tid; e < n * n * 32; e += kThreads) ou[e] = 0.f;
  __syncthreads();
  if (warp == 0) {
    const float r = (lane < NT) ? root[lane] : ninf();
    const float rm = warp_max(r);
    ou[(size_t)(n - 1) * 32 + lane] = (lane < NT && rm != ninf()) ? fexp(r - rm) : 0.f;
    if (lane == 0) osc[n - 1] = (rm == ninf()) ? ninfd() : (double)rm;
  }
  __syncthreads();
  float* REs = smf;                  // [3][32 A][kBS][32 C]
  float* Os = smf + 3 * kBS * 1024;  // [kMaxN parents][32 A]
  for (int w = n; w >= 2; --w) {
    const int nsp = n - w + 1;
    const int nslot = (w == 2) ? 1 : 3;
    // stage parent outside vectors (with the parent's own sticky folded into its scale)
    for (int e = tid; e < nsp * 32; e += kThreads) {
      const int s = e >> 5, A = e & 31;
      Os[e] = (A < NT) ? ou[(size_t)(s * n + s + w - 1) * 32 + A] : 0.f;
    }
    // ---- Q-build: Q[s][slot][B][C] = sum_A o_s[A] R_t[A, B', C'] (lane = C)
    for (int b0 = 0; b0 < 32; b0 += kBS) {
      // REs[sl][A][bb][C]: 512 B contiguous per (sl, A)
      for (int e = tid; e < nslot * 32 * 32; e += kThreads) {
        const int sl = e >> 10, r = e & 1023;
        const int A = r >> 5, q = r & 31;
        const int t = slot_type(sl, w);
        cpa16(REs + (sl * 32 + A) * kBS * 32 + 4 * q, RE + (((size_t)t * 32 + A) * 32 + b0) * 32 + 4 * q);
      }
      cpa_commit_wait();
      __syncthreads();
      for (int sl = 0; sl < nslot; ++sl) {
        float q4[kSpW][kBS];
#pragma unroll
        for (int q = 0; q < kSpW; ++q)
#pragma unroll
          for (int bb = 0; bb < kBS; ++bb) q4[q][bb] = 0.f;
        for (int A = 0; A < NT; ++A) {
          float rr[kBS];
#pragma unroll
          for (int bb = 0; bb < kBS; ++bb) rr[bb] = REs[((sl * 32 + A) * kBS + bb) * 32 + lane];
#pragma unroll
          for (int q = 0; q < kSpW; ++q) {
            const int s = warp + q * kWarps;
            if (s < nsp) {
              const float o = Os[s * 32 + A];
#pragma unroll
              for (int bb = 0; bb < kBS; ++bb) q4[q][bb] = fmaf(o, rr[bb], q4[q][bb]);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < kSpW; ++q) {
          const int s = warp + q * kWarps;
          if (s < nsp) {
#pragma unroll
            for (int bb = 0; bb < kBS; ++bb) {
              Pw[(size_t)s * 3 * 1024 + sl * 1024 + (b0 + bb) * 32 + lane] = q4[q][bb];  // [B][C]
              Q2[(size_t)s * 3 * 1024 + sl * 1024 + lane * 32 + (b0 + bb)] = q4[q][bb];  // [C][B]
            }
          }
        }
      }
      __syncthreads();
    }
    // ---- pushes; parent scale = osc + sticky (constituency.py:303)
    for (int side = 0; side < 2; ++side) {
      for (int s = warp; s < nsp; s += kWarps) {
        const int i = s, j = i + w - 1;
        const double ps = osc[i * n + j] + (double)STK(i, j);
        if (ps == ninfd()) continue;
        for (int k = i; k < j; ++k) {
          const int sl = (w == 2) ? 0 : (k == i ? 1 : (k == j - 1 ? 2 : 0));
          // side 0: left child (i,k) gets sum_C Q[B][C] u_(k+1)j[C];  side 1: right child (k+1,j)
          const int si = side == 0 ? k + 1 : i, sj = side == 0 ? j : k;  // sibling span
          const int ci = side == 0 ? i : k + 1, cj = side == 0 ? k : j;  // child span
          const double sib = isc[si * n + sj];
          if (sib == ninfd()) continue;
          const float sv = iu[(size_t)(si * n + sj) * 32 + lane];
          float g = 0.f;
          const float* Qm = (side == 0 ? Q2 : Pw) + (size_t)s * 3 * 1024 + sl * 1024;  // [lane-major row][x]
#pragma unroll 8
          for (int x = 0; x < 32; ++x) {
            const float svx = __shfl_sync(0xffffffffu, sv, x);
            g = fmaf(Qm[x * 32 + lane], svx, g);
          }
          // normalise the contribution (keeps the child's vector O(1) at any depth)
          const float gm = warp_max(g);
          if (!(gm > 0.f)) continue;
          g = g / gm;
          // merge contribution (scale cs, vec g) into child
          const double cs = ps + sib + (double)flog(gm);
          const size_t co = (size_t)(ci * n + cj);
          const double old = osc[co];
          const double M = fmax(old, cs);
          const float a1 = (old == ninfd()) ? 0.f : fexp((float)(old - M));
          const float a2 = fexp((float)(cs - M));
          ou[co * 32 + lane] = ou[co * 32 + lane] * a1 + g * a2;
          __syncwarp();
          if (lane == 0) osc[co] = M;
          __syncwarp();
        }
      }
      __syncthreads();
    }
  }
  // ---- span marginals (constituency.py:334-338)
  for (int e = warp; e < n * n; e += kWarps) {
    const int i = e / n, j = e - i * n;
    float v = 0.f;
    if (i <= j) {
      const double si = isc[e], so = osc[e];
      const float p = ou[(size_t)e * 32 + lane] * iu[(size_t)e * 32 + lane];
      const float tot = warp_sum(p);
      if (si != ninfd() && so != ninfd() && tot > 0.f) v = fexp((float)(si + so - Z)) * tot;
    }
    if (lane == 0) mg[e] = v;
  }
}

int pcfg_check(int64_t B, int n, int NT, int PT) {
  if (B < 0 || n < 1 || NT < 1 || PT < 1) return SDB_ERR_ARG;
  if (n > kMaxN || NT > 32 || PT > 32) return SDB_ERR_UNSUPPORTED;
  return SDB_OK;
}

}  // namespace

extern "C" size_t sdb_pcfg_fb_workspace(int64_t B, int32_t n, int32_t NT, int32_t PT) {
  size_t bytes = 0;
  pcfg_carve(nullptr, B, n, NT, PT, &bytes);
  return bytes;
}

extern "C" int sdb_pcfg_fb(const float* root, const float* rules, const float* emissions, const float* sticky,
                           int64_t B, int32_t n, int32_t NT, int32_t PT, double* logz, float* span_marg,
                           int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  int rc = pcfg_check(B, n, NT, PT);
  if (rc) return rc;
  if (!root || !rules || !emissions || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  size_t need = 0;
  PcfgWs ws = pcfg_carve(workspace, B, n, NT, PT, &need);
  if (!workspace || ws_bytes < need) return SDB_ERR_WORKSPACE;
  const size_t smem = (size_t)(3 * kBS * 1024 + kMaxN * 3 * kBS * 32) * 4;
  cudaStream_t s = (cudaStream_t)stream;
  if (span_marg) {
    if (cudaFuncSetAttribute(pcfg_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SDB_ERR_CUDA;
    pcfg_kernel<true><<<(unsigned)B, kThreads, smem, s>>>(root, rules, emissions, sticky, n, NT, PT, ws, logz,
                                                          span_marg, status);
  } else {
    if (cudaFuncSetAttribute(pcfg_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SDB_ERR_CUDA;
    pcfg_kernel<false><<<(unsigned)B, kThreads, smem, s>>>(root, rules, emissions, sticky, n, NT, PT, ws, logz,
                                                           nullptr, status);
  }
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
