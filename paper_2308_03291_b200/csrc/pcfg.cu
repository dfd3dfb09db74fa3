// PCFG (Chomsky normal form): inside log-partition and constituent (span)
// marginals via inside/outside in scaled linear space; max-plus argmax.
//
// Reference: structdist constituency.py:246-371 (_pcfg_inside, pcfg_inside,
// pcfg_gradients, _pcfg_walk, pcfg_argmax).  Per instance: root [NT],
// binary_rules [NT][S][S] (children: NTs 0..NT-1 then PTs NT..S-1),
// emissions [n][PT], optional sticky [n][n] in {0,-inf}.  This kernel
// serves NT, PT <= 32, n <= 64 (the C5b shape); larger grammars / sentences
// take the general fp64 path in pcfg_gen.cu.
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

size_t pcfg_gen_workspace(int64_t B, int n, int NT, int PT, bool grad);
int pcfg_gen_launch(int mode, const float* root, const float* rules, const float* emissions, const float* sticky,
                    int64_t B, int n, int NT, int PT, double* logz, float* span_marg, float* groot, float* grules,
                    float* gemis, int32_t* status, void* workspace, size_t ws_bytes, cudaStream_t s);

namespace {

constexpr int kThreads = 256;  // pcfg_max_kernel
constexpr int kWarps = kThreads / 32;
constexpr int kPT = 512;       // pcfg_kernel: 16 warps (<= 128 registers) for latency hiding
constexpr int kPWarps = kPT / 32;
constexpr int kSpW = 4;    // spans per warp (register block); n <= 64 = kSpW * kPWarps
constexpr int kBS = 4;     // B-slice width
constexpr int kMaxN = 64;
constexpr int kCP = 8;     // outside parents per shared-memory chunk
static_assert(kPWarps == 2 * kCP && kSpW * kPWarps >= 64, "pcfg_kernel warp roles");

struct PcfgWs {
  float* RE;    // [B][4][32 A][32 B][32 C]  exp(rules) per child-class block t, zero padded
  float* RT;    // [B][4][32 B][32 C][32 A]  the same, A fastest (inside contraction)
  float* iu;    // [B][n][n][32]
  double* isc;  // [B][n][n]
  float* ou;    // [B][n][n][32]
  double* osc;  // [B][n][n]
  float* P;     // [B][n][3][32][32] per-width scratch (P in inside, Q in outside)
  float* P2;    // [B][n][3][32][32] inside pair products recomputed in the outside pass (mode 2)
  float* G;     // [B][4][32 A][32 B][32 C] expected rule counts before the exp(rule) factor (mode 2)
};

PcfgWs pcfg_carve(void* base, int64_t B, int n, int NT, int PT, size_t* bytes, bool grad = false) {
  (void)NT;
  (void)PT;
  Carve c(base);
  PcfgWs w;
  w.RE = c.take<float>((size_t)B * 4 * 32768);  // REp[t][A][B][C] zero-padded per child block
  w.RT = c.take<float>((size_t)B * 4 * 32768);  // RTp[t][B][C][A]
  w.iu = c.take<float>((size_t)B * n * n * 32);
  w.isc = c.take<double>((size_t)B * n * n);
  w.ou = c.take<float>((size_t)B * n * n * 32);
  w.osc = c.take<double>((size_t)B * n * n);
  w.P = c.take<float>((size_t)B * n * 3 * 1024);
  w.P2 = grad ? c.take<float>((size_t)B * n * 3 * 1024) : nullptr;
  w.G = grad ? c.take<float>((size_t)B * 4 * 32768) : nullptr;
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

// inner[q] += sum_{slot, bb, C} R_t[A = lane][B'][C'] P[s_q][slot][bb][C] for the QN spans
// s_q = warp + q kPWarps of this warp (one B-slice of the inside contraction)
template <int QN>
__device__ __forceinline__ void contract_slice(const float* __restrict__ RTs, const float* __restrict__ Ps, int nslot,
                                               int warp, int lane, float* inner) {
  for (int sl = 0; sl < nslot; ++sl) {
    for (int bb = 0; bb < kBS; ++bb) {
#pragma unroll 4
      for (int C = 0; C < 32; C += 4) {
        const float r0 = RTs[((sl * kBS + bb) * 32 + C + 0) * 32 + lane];
        const float r1 = RTs[((sl * kBS + bb) * 32 + C + 1) * 32 + lane];
        const float r2 = RTs[((sl * kBS + bb) * 32 + C + 2) * 32 + lane];
        const float r3 = RTs[((sl * kBS + bb) * 32 + C + 3) * 32 + lane];
#pragma unroll
        for (int q = 0; q < QN; ++q) {
          const int sp = warp + q * kPWarps;
          const float4 p = *reinterpret_cast<const float4*>(&Ps[((sp * 3 + sl) * kBS + bb) * 32 + C]);
          inner[q] = fmaf(r0, p.x, fmaf(r1, p.y, fmaf(r2, p.z, fmaf(r3, p.w, inner[q]))));
        }
      }
    }
  }
}

// child class offsets of block t: t0 = (NT,NT) t1 = (PT,NT) t2 = (NT,PT) t3 = (PT,PT)
__device__ __forceinline__ int boff(int t, int NT) { return (t == 1 || t == 3) ? NT : 0; }
__device__ __forceinline__ int coff(int t, int NT) { return (t == 2 || t == 3) ? NT : 0; }
__device__ __forceinline__ int bcnt(int t, int NT, int PT) { return (t == 1 || t == 3) ? PT : NT; }
__device__ __forceinline__ int ccnt(int t, int NT, int PT) { return (t == 2 || t == 3) ? PT : NT; }
// block of slot `sl` at width w: w == 2 -> only slot 0 = t3; else slot 0 = t0 (interior), 1 = t1 (k=i), 2 = t2 (k=j-1)
__device__ __forceinline__ int slot_type(int sl, int w) { return w == 2 ? 3 : sl; }

struct PcfgGradOut {
  float* root;   // [B][NT]
  float* rules;  // [B][NT][S][S]
  float* emis;   // [B][n][PT]
};

// kMode: 0 = log Z, 1 = + span marginals, 2 = + rule / root / emission
// expected counts (the full pcfg_gradients, constituency.py:292-340)
template <int kMode>
__global__ void __launch_bounds__(kPT, 1) pcfg_kernel(
    const float* __restrict__ root_all, const float* __restrict__ rules_all, const float* __restrict__ emis_all,
    const float* __restrict__ sticky_all, int n, int NT, int PT, PcfgWs ws, double* __restrict__ logz,
    float* __restrict__ marg_all, PcfgGradOut gout, int32_t* __restrict__ status) {
  constexpr bool kMarg = kMode >= 1;
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
  __shared__ int badsh;
  __shared__ double smax_s[kMaxN];
  __shared__ double smax2_s[kMaxN];
  __shared__ __align__(16) float svs[kPWarps][2][32];  // per-warp sibling vectors (push dot products)
  __shared__ __align__(16) float lvs[kPWarps][4][32];  // per-warp left-child vectors (P-build)
  float* P2 = kMode == 2 ? ws.P2 + (size_t)b * n * 3 * 1024 : nullptr;
  float* G = kMode == 2 ? ws.G + (size_t)b * 4 * 32768 : nullptr;
  if (tid == 0) badsh = 0;
  __syncthreads();
  auto STK = [&](int i, int j) -> float { return sticky ? sticky[i * n + j] : 0.f; };

  // ---- prologue: exp(rules) into zero-padded per-block layouts (RE: C fastest, RT: A fastest),
  // input checks
  {
    int bad = 0;
    for (int e = tid; e < NT * S * S; e += kPT) bad |= bad_input(rules[e]);
    for (int e = tid; e < 4 * 32768; e += kPT) {
      const int t = e >> 15, r = e & 32767;
      const int A = r >> 10, Bi = (r >> 5) & 31, C = r & 31;
      float v = 0.f;
      if (A < NT && Bi < bcnt(t, NT, PT) && C < ccnt(t, NT, PT))
        v = fexp(rules[((size_t)A * S + boff(t, NT) + Bi) * S + coff(t, NT) + C]);
      RE[e] = v;                                              // [t][A][B][C]
      RT[(((size_t)t * 32 + Bi) * 32 + C) * 32 + A] = v;      // [t][B][C][A]
    }
    for (int e = tid; e < NT; e += kPT) bad |= bad_input(root[e]);
    for (int e = tid; e < n * PT; e += kPT) bad |= bad_input(emis[e]);
    if (sticky)
      for (int e = tid; e < n * n; e += kPT) bad |= !(sticky[e] == 0.f || sticky[e] == ninf());
    if (bad) atomicOr(&badsh, 1);
    if (kMode == 2)
      for (int e = tid; e < 4 * 32768; e += kPT) G[e] = 0.f;
  }
  __syncthreads();
  // ---- width 1: preterminal slots (constituency.py:257-258)
  for (int i = warp; i < n; i += kPWarps) {
    const float x = (lane < PT) ? emis[i * PT + lane] : ninf();
    const float m = warp_max(x);
    const float st = STK(i, i);
    const bool dead = (m == ninf()) || st == ninf();
    iu[(size_t)(i * n + i) * 32 + lane] = dead ? 0.f : fexp(x - m);
    if (lane == 0) isc[i * n + i] = dead ? ninfd() : (double)m;
  }
  __syncthreads();

  // P-build for all spans of width w (warp per span): P_t[B][C] = sum_k f_k u_ik[B] u_(k+1)j[C],
  // f_k = exp(s_ik + s_(k+1)j - Smax); Smax -> smx[i]
  auto pbuild = [&](int w, float* dst, double* smx) {
    const int nsp = n - w + 1;
    for (int i = warp; i < nsp; i += kPWarps) {
      const int j = i + w - 1;
      double sm = ninfd();
      for (int k = i + lane; k < j; k += 32) sm = fmax(sm, isc[i * n + k] + isc[(k + 1) * n + j]);
      sm = warp_maxd(sm);
      if (lane == 0) smx[i] = sm;
      // slot 0: the interior splits (both children wide); at w == 2 the single split (PT, PT)
      float acc[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) acc[q] = 0.f;
      const int klo = (w == 2) ? i : i + 1, khi = (w == 2) ? j : j - 1;
      if (sm != ninfd()) {
        // four splits per pass: their (L2-resident) chart loads are all issued before the
        // shuffle/FMA work, so one L2 latency is exposed per pass instead of per split
        for (int k0 = klo; k0 < khi; k0 += 4) {
          double sk[4];
          float lv[4], rv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int k = min(k0 + u, khi - 1);
            sk[u] = (k0 + u < khi) ? isc[i * n + k] + isc[(k + 1) * n + j] : ninfd();
            lv[u] = iu[(size_t)(i * n + k) * 32 + lane];
            rv[u] = iu[(size_t)((k + 1) * n + j) * 32 + lane];  // lane = C
          }
          // the left vectors go through a per-warp shared slot, read back as 16-byte broadcasts
          // (8 LDS.128 per split instead of 32 shuffles)
#pragma unroll
          for (int u = 0; u < 4; ++u) lvs[warp][u][lane] = lv[u];
          __syncwarp();
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (sk[u] == ninfd()) continue;
            const float rf = rv[u] * fexp((float)(sk[u] - sm));
            const float4* l4 = reinterpret_cast<const float4*>(lvs[warp][u]);
#pragma unroll
            for (int q4 = 0; q4 < 8; ++q4) {
              const float4 lb = l4[q4];
              acc[4 * q4 + 0] = fmaf(lb.x, rf, acc[4 * q4 + 0]);
              acc[4 * q4 + 1] = fmaf(lb.y, rf, acc[4 * q4 + 1]);
              acc[4 * q4 + 2] = fmaf(lb.z, rf, acc[4 * q4 + 2]);
              acc[4 * q4 + 3] = fmaf(lb.w, rf, acc[4 * q4 + 3]);
            }
          }
          __syncwarp();  // the slots are rewritten by the next pass
        }
      }
      float* pp = dst + (size_t)i * 3 * 1024;
#pragma unroll
      for (int q = 0; q < 32; ++q) pp[q * 32 + lane] = acc[q];  // [slot 0][B][C]
      // slots 1 (k = i: (PT, NT)) and 2 (k = j-1: (NT, PT)) hold ONE split each: rank-1
      // outer products written directly (no accumulator registers)
      if (w > 2) {
#pragma unroll 1
        for (int e = 0; e < 2; ++e) {
          const int k = e == 0 ? i : j - 1;
          const double skk = isc[i * n + k] + isc[(k + 1) * n + j];
          const bool live = (sm != ninfd()) && (skk != ninfd());
          const float rf = live ? iu[(size_t)((k + 1) * n + j) * 32 + lane] * fexp((float)(skk - sm)) : 0.f;
          lvs[warp][0][lane] = iu[(size_t)(i * n + k) * 32 + lane];
          __syncwarp();
          const float4* l4 = reinterpret_cast<const float4*>(lvs[warp][0]);
          float* pe = pp + (1 + e) * 1024;
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            const float4 lb = l4[q4];
            pe[(4 * q4 + 0) * 32 + lane] = lb.x * rf;
            pe[(4 * q4 + 1) * 32 + lane] = lb.y * rf;
            pe[(4 * q4 + 2) * 32 + lane] = lb.z * rf;
            pe[(4 * q4 + 3) * 32 + lane] = lb.w * rf;
          }
          __syncwarp();
        }
      }
    }
  };

  float* RTs = smf;                 // [3][kBS][32 C][32 A]
  float* Ps = smf + 3 * kBS * 1024; // [kMaxN spans][3][kBS][32 C]

  // ================================================================ inside
  for (int w = 2; w <= n; ++w) {
    const int nsp = n - w + 1;
    const int nslot = (w == 2) ? 1 : 3;
    // ---- P-build: warp per span
    pbuild(w, Pw, smax_s);
    __syncthreads();
    // ---- contraction: inner[s][A] = sum_{slot,B,C} R_t[A,B',C'] P[s][slot][B][C]
    float inner[kSpW];
#pragma unroll
    for (int q = 0; q < kSpW; ++q) inner[q] = 0.f;
    for (int b0 = 0; b0 < 32; b0 += kBS) {
      // stage R slice RTs[sl][bb][C][A] (4 KB contiguous per (sl, bb)) and the P slice
      // Ps[s][sl][bb][C] (512 B contiguous per (s, sl)) with 16-byte cp.async
      for (int e = tid; e < nslot * kBS * 256; e += kPT) {
        const int sl = e / (kBS * 256), r = e - sl * (kBS * 256);
        const int t = slot_type(sl, w);
        cpa16(RTs + sl * kBS * 1024 + 4 * r, RT + ((size_t)t * 32 + b0) * 1024 + 4 * r);
      }
      for (int e = tid; e < nsp * nslot * 32; e += kPT) {
        const int s2 = e / (nslot * 32), r = e - s2 * (nslot * 32);
        const int sl = r >> 5, q = r & 31;
        cpa16(Ps + (s2 * 3 + sl) * kBS * 32 + 4 * q, Pw + (size_t)s2 * 3 * 1024 + sl * 1024 + b0 * 32 + 4 * q);
      }
      cpa_commit_wait();
      __syncthreads();
      // the warp's span count qn is warp-uniform: dispatch to a body with exactly qn spans so
      // wide widths (few spans) do not issue the idle span slots
      const int qn = nsp > warp ? min(kSpW, (nsp - warp + kPWarps - 1) / kPWarps) : 0;
      switch (qn) {
        case 8: contract_slice<8>(RTs, Ps, nslot, warp, lane, inner); break;
        case 7: contract_slice<7>(RTs, Ps, nslot, warp, lane, inner); break;
        case 6: contract_slice<6>(RTs, Ps, nslot, warp, lane, inner); break;
        case 5: contract_slice<5>(RTs, Ps, nslot, warp, lane, inner); break;
        case 4: contract_slice<4>(RTs, Ps, nslot, warp, lane, inner); break;
        case 3: contract_slice<3>(RTs, Ps, nslot, warp, lane, inner); break;
        case 2: contract_slice<2>(RTs, Ps, nslot, warp, lane, inner); break;
        case 1: contract_slice<1>(RTs, Ps, nslot, warp, lane, inner); break;
        default: break;
      }
      __syncthreads();
    }
    // ---- normalise and store the width's cells (constituency.py:264-265)
#pragma unroll
    for (int q = 0; q < kSpW; ++q) {
      const int i = warp + q * kPWarps;
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
  const int S2 = S * S;
  if (Z == ninfd() || badsh) {
    for (int e = tid; e < n * n; e += kPT) mg[e] = 0.f;
    if (kMode == 2) {
      for (int e = tid; e < NT; e += kPT) gout.root[(size_t)b * NT + e] = 0.f;
      for (int e = tid; e < NT * S2; e += kPT) gout.rules[(size_t)b * NT * S2 + e] = 0.f;
      for (int e = tid; e < n * PT; e += kPT) gout.emis[(size_t)b * n * PT + e] = 0.f;
    }
    return;
  }

  // =============================================================== outside
  for (int e = tid; e < n * n; e += kPT) osc[e] = ninfd();
  for (int e = tid; e < n * n * 32; e += kPT) ou[e] = 0.f;
  __syncthreads();
  if (warp == 0) {
    const float r = (lane < NT) ? root[lane] : ninf();
    const float rm = warp_max(r);
    ou[(size_t)(n - 1) * 32 + lane] = (lane < NT && rm != ninf()) ? fexp(r - rm) : 0.f;
    if (lane == 0) osc[n - 1] = (rm == ninf()) ? ninfd() : (double)rm;
  }
  __syncthreads();
  float* REs = smf;                                  // [2][3][32 A][kBS][32 C] (double buffer)
  float* Os = REs + 2 * 3 * kBS * 1024;              // [32 A][kCP parents]
  float* Qc = Os + kCP * 32;                         // [kCP][3][32 B][33 C] (padded rows: both push
                                                     //  orientations read it conflict-free)
  for (int w = n; w >= 2; --w) {
    const int nsp = n - w + 1;
    const int nslot = (w == 2) ? 1 : 3;
    if (kMode == 2) {
      // expected rule counts of the width's parents (constituency.py:312-314):
      // G_t[A][B][C] += exp(o_s + sticky_s + Smax_s - Z) o_s[A] P_s[t][B][C]; exp(rule) applied at the end
      float* Cs = smf + 3 * kBS * 1024 + kMaxN * 3 * kBS * 32;  // [nsp][32 A]
      pbuild(w, P2, smax2_s);
      __syncthreads();
      for (int e = tid; e < nsp * 32; e += kPT) {
        const int s2 = e >> 5, A = e & 31, i = s2, j = s2 + w - 1;
        const double c = osc[i * n + j] + (double)STK(i, j) + smax2_s[s2] - Z;
        Cs[e] = (A < NT && c != ninfd()) ? (float)(exp(c) * (double)ou[(size_t)(i * n + j) * 32 + A]) : 0.f;
      }
      __syncthreads();
      for (int sl = 0; sl < nslot; ++sl) {
        float* Gt = G + (size_t)slot_type(sl, w) * 32768;
        for (int r = 0; r < 1024 / kPT; ++r) {
          const int bc = tid + kPT * r;
          float acc[32];
#pragma unroll
          for (int A = 0; A < 32; ++A) acc[A] = 0.f;
          for (int s2 = 0; s2 < nsp; ++s2) {
            const float pv = P2[(size_t)s2 * 3 * 1024 + sl * 1024 + bc];
            if (pv == 0.f) continue;
#pragma unroll
            for (int A = 0; A < 32; ++A) acc[A] = fmaf(Cs[s2 * 32 + A], pv, acc[A]);
          }
          for (int A = 0; A < NT; ++A) Gt[A * 1024 + bc] += acc[A];
        }
      }
      __syncthreads();
    }
    // Parents are processed in chunks of kCP: their Q matrices are built straight
    // into shared memory (both orientations) and the pushes read them there --
    // no global scratch round trip, each Q row is read from smem by every split
    // of its parent.
    for (int c0 = 0; c0 < nsp; c0 += kCP) {
      const int cn = min(kCP, nsp - c0);
      // stage the chunk's parent outside vectors
      for (int e = tid; e < cn * 32; e += kPT) {
        const int pz = e >> 5, A = e & 31, s = c0 + pz;
        Os[A * kCP + pz] = (A < NT) ? ou[(size_t)(s * n + s + w - 1) * 32 + A] : 0.f;  // [A][parent]
      }
      // ---- Q-build: Q[p][slot][B][C] = sum_A o_p[A] R_t[A, B', C'] (warp = parent, lane = C);
      // R slices double-buffered through shared memory
      auto stage = [&](int b0, float* dst) {
        for (int e = tid; e < nslot * 32 * 32; e += kPT) {
          const int sl = e >> 10, r = e & 1023;
          const int A = r >> 5, q = r & 31;
          const int t = slot_type(sl, w);
          cpa16(dst + (sl * 32 + A) * kBS * 32 + 4 * q, RE + (((size_t)t * 32 + A) * 32 + b0) * 32 + 4 * q);
        }
        asm volatile("cp.async.commit_group;\n" ::);
      };
      stage(0, REs);
      for (int b0 = 0; b0 < 32; b0 += kBS) {
        float* cur = REs + ((b0 / kBS) & 1) * 3 * kBS * 1024;
        if (b0 + kBS < 32) {
          stage(b0 + kBS, REs + (((b0 / kBS) + 1) & 1) * 3 * kBS * 1024);
          asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
          asm volatile("cp.async.wait_group 0;\n" ::);
        }
        __syncthreads();
        // register-tiled: thread = (2 parents, 3 slots) x one (bb, C) column, so every R word
        // loaded from shared memory feeds 2 FMAs and every parent weight 3
        {
          static_assert(kCP == 8 && kPT == 512 && kBS * 32 == 128, "Q-build tiling");
          const int pg = tid >> 7, c = tid & 127;  // parents 2pg, 2pg+1 (warp-uniform), column c
          if (2 * pg < cn) {
            float q[2][3];
#pragma unroll
            for (int pp = 0; pp < 2; ++pp)
#pragma unroll
              for (int sl = 0; sl < 3; ++sl) q[pp][sl] = 0.f;
            for (int A = 0; A < NT; ++A) {
              float r[3];
              const float2 o2 = *reinterpret_cast<const float2*>(&Os[A * kCP + 2 * pg]);
              const float o[2] = {o2.x, o2.y};
#pragma unroll
              for (int sl = 0; sl < 3; ++sl) r[sl] = sl < nslot ? cur[(sl * 32 + A) * 128 + c] : 0.f;
#pragma unroll
              for (int pp = 0; pp < 2; ++pp)
#pragma unroll
                for (int sl = 0; sl < 3; ++sl) q[pp][sl] = fmaf(o[pp], r[sl], q[pp][sl]);
            }
            const int bb = c >> 5, C = c & 31;
#pragma unroll
            for (int pp = 0; pp < 2; ++pp)
#pragma unroll
              for (int sl = 0; sl < 3; ++sl)
                if (2 * pg + pp < cn && sl < nslot)
                  Qc[(((2 * pg + pp) * 3 + sl) * 32 + b0 + bb) * 33 + C] = q[pp][sl];  // [B][C]
          }
        }
        __syncthreads();
      }
      // ---- pushes; parent scale = osc + sticky (constituency.py:303)
      for (int side = 0; side < 2; ++side) {
        // two warps per parent (kPWarps = 2 kCP): warp half h takes the split pairs
        // (k, k+1), k = i + 2h (mod 4) -- the children of distinct splits are distinct
        const int half = warp / kCP;
        for (int pz = warp % kCP; pz < cn; pz += kCP) {
          const int s = c0 + pz;
          const int i = s, j = i + w - 1;
          const double ps = osc[i * n + j] + (double)STK(i, j);
          if (ps == ninfd()) continue;
          // split k's loads (sibling inside scale/vector, child outside state) are issued one
          // split ahead, so their global latency overlaps the previous split's dot product
          // (children and siblings of one parent's splits are all distinct spans)
          auto span_of = [&](int k, int& si, int& sj, size_t& co) {
            // side 0: left child (i,k) gets sum_C Q[B][C] u_(k+1)j[C];  side 1: right child (k+1,j)
            si = side == 0 ? k + 1 : i;
            sj = side == 0 ? j : k;  // sibling span
            const int ci = side == 0 ? i : k + 1, cj = side == 0 ? k : j;  // child span
            co = (size_t)(ci * n + cj);
          };
          // two splits per pass (independent children: their dot products and merges
          // interleave), the next pass's loads issued before this pass's arithmetic
          struct Item { double sib, old; float sv, ou; size_t co; };
          auto fetch = [&](int k, Item& x) {
            int si, sj;
            span_of(k, si, sj, x.co);
            x.sib = isc[si * n + sj];
            x.old = osc[x.co];
            x.sv = iu[(size_t)(si * n + sj) * 32 + lane];
            x.ou = ou[x.co * 32 + lane];
          };
          auto slot_of = [&](int k) { return (w == 2) ? 0 : (k == i ? 1 : (k == j - 1 ? 2 : 0)); };
          auto dot = [&](int k, const float* sv4) {
            const float* Qm = Qc + (size_t)(pz * 3 + slot_of(k)) * 32 * 33;
            const float4* s4 = reinterpret_cast<const float4*>(sv4);
            float g = 0.f, g2 = 0.f;
            if (side == 0) {  // lane = B: row B of Q
#pragma unroll
              for (int x4 = 0; x4 < 8; ++x4) {
                const float4 v = s4[x4];
                g = fmaf(Qm[lane * 33 + 4 * x4 + 0], v.x, g);
                g2 = fmaf(Qm[lane * 33 + 4 * x4 + 1], v.y, g2);
                g = fmaf(Qm[lane * 33 + 4 * x4 + 2], v.z, g);
                g2 = fmaf(Qm[lane * 33 + 4 * x4 + 3], v.w, g2);
              }
            } else {          // lane = C: column C of Q
#pragma unroll
              for (int x4 = 0; x4 < 8; ++x4) {
                const float4 v = s4[x4];
                g = fmaf(Qm[(4 * x4 + 0) * 33 + lane], v.x, g);
                g2 = fmaf(Qm[(4 * x4 + 1) * 33 + lane], v.y, g2);
                g = fmaf(Qm[(4 * x4 + 2) * 33 + lane], v.z, g);
                g2 = fmaf(Qm[(4 * x4 + 3) * 33 + lane], v.w, g2);
              }
            }
            return g + g2;
          };
          // merge contribution g (child scale ps + sib + log max g) into the child
          auto merge = [&](const Item& x, float g) {
            if (x.sib == ninfd()) return;
            // g >= 0: its float bits order like unsigned ints -> one REDUX instead of 5 shuffles
            const float gm = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(g)));
            if (!(gm > 0.f)) return;
            const double cs = ps + x.sib + (double)flog(gm);
            const double M = fmax(x.old, cs);
            const float a1 = (x.old == ninfd()) ? 0.f : fexp((float)(x.old - M));
            const float a2 = fexp((float)(cs - M));
            ou[x.co * 32 + lane] = x.ou * a1 + (g / gm) * a2;
            if (lane == 0) osc[x.co] = M;  // this child is not touched again in this side pass
          };
          Item A, Bv;
          const int kf = i + 2 * half;
          if (kf < j) fetch(kf, A);
          if (kf + 1 < j) fetch(kf + 1, Bv);
          for (int k = kf; k < j; k += 4) {
            const Item a = A, bq = Bv;
            const bool hb = k + 1 < j;
            if (k + 4 < j) fetch(k + 4, A);
            if (k + 5 < j) fetch(k + 5, Bv);
            // the sibling vectors go through per-warp shared slots and are read back as
            // 16-byte broadcasts (8 LDS.128 instead of 32 shuffles per dot product)
            svs[warp][0][lane] = a.sv;
            svs[warp][1][lane] = hb ? bq.sv : 0.f;
            __syncwarp();
            const float ga = dot(k, svs[warp][0]);
            const float gb = hb ? dot(k + 1, svs[warp][1]) : 0.f;
            __syncwarp();  // the slots are rewritten by the next pass
            merge(a, ga);
            if (hb) merge(bq, gb);
          }
        }
        __syncthreads();
      }
    }
  }
  // ---- span marginals (constituency.py:334-338)
  for (int e = warp; e < n * n; e += kPWarps) {
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
  if (kMode != 2) return;
  __syncthreads();
  // root gradient exp(root + chart[0,n-1] - Z) (constituency.py:326)
  if (warp == 0 && lane < NT) {
    const double si = isc[n - 1];
    const float u = iu[(size_t)(n - 1) * 32 + lane];
    gout.root[(size_t)b * NT + lane] =
        (si == ninfd() || !(u > 0.f)) ? 0.f : (float)(exp((double)root[lane] + si - Z) * (double)u);
  }
  // emission gradient exp(outside[i,i,PT] + sticky[i,i] + emissions - Z) (constituency.py:327-329)
  for (int i = warp; i < n; i += kPWarps) {
    const int e = i * n + i;
    const double c = osc[e] + (double)STK(i, i) + isc[e] - Z;
    const float v = ou[(size_t)e * 32 + lane] * iu[(size_t)e * 32 + lane];
    if (lane < PT) gout.emis[((size_t)b * n + i) * PT + lane] = (c == ninfd() || !(v > 0.f)) ? 0.f : (float)(exp(c) * (double)v);
  }
  // rule gradient = G_t[A][B'][C'] * exp(rules[A][B][C])
  for (int e = tid; e < NT * S2; e += kPT) {
    const int A = e / S2, r = e - A * S2, Bf = r / S, Cf = r - Bf * S;
    const int t = (Bf < NT ? 0 : 1) + (Cf < NT ? 0 : 2);
    const int Bi = Bf - boff(t, NT), Ci = Cf - coff(t, NT);
    const size_t gi = (size_t)t * 32768 + ((size_t)A * 32 + Bi) * 32 + Ci;
    gout.rules[(size_t)b * NT * S2 + e] = G[gi] * RE[gi];
  }
}


// ================================================================ max-plus
// fp64 max-plus chart (constituency.py:246-266 with reduce = max, exact sums
// in the reference's order) and the top-down derivation walk
// (constituency.py:343-371): first-maximum picks over the root symbols and
// over the flattened (split, left symbol, right symbol) candidates.
struct ArgBest {
  double v;
  int i;
};
__device__ __forceinline__ ArgBest arg_better(ArgBest a, ArgBest b) {
  return (b.v > a.v || (b.v == a.v && b.i < a.i)) ? b : a;
}
__device__ ArgBest block_argmax(ArgBest x, ArgBest* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgBest y;
    y.v = __shfl_xor_sync(0xffffffffu, x.v, o);
    y.i = __shfl_xor_sync(0xffffffffu, x.i, o);
    x = arg_better(x, y);
  }
  if (lane == 0) red[warp] = x;
  __syncthreads();
  ArgBest r = red[0];
  for (int q = 1; q < (int)(blockDim.x >> 5); ++q) r = arg_better(r, red[q]);
  __syncthreads();
  return r;
}

// kLog: log-semiring chart (constituency.py:246-266 with logsumexp) and
// Gumbel-max picks from the caller's stream (pcfg_sample, constituency.py:374-378);
// mask [B][num][n][n], used [B].
template <bool kLog, typename TP = float>  // TP = double: the exact mode (float64 grammar)
__global__ void __launch_bounds__(kThreads) pcfg_max_kernel(
    const TP* __restrict__ root_all, const TP* __restrict__ rules_all, const TP* __restrict__ emis_all,
    const TP* __restrict__ sticky_all, int n, int NT, int PT, double* __restrict__ chart_all,
    int8_t* __restrict__ mask_all, double* __restrict__ score, int32_t* __restrict__ status,
    const double* __restrict__ noise_all = nullptr, int64_t cap = 0, int num = 1, int32_t* __restrict__ used = nullptr) {
  extern __shared__ double pairs[];  // [S][S], then the walk stack [3][2n] ints
  __shared__ ArgBest red[kWarps];
  __shared__ int badsh;
  const int S = NT + PT, S2 = S * S;
  int* stk_i = reinterpret_cast<int*>(pairs + S2);
  int* stk_j = stk_i + 2 * n;
  int* stk_a = stk_j + 2 * n;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const TP* root = root_all + (size_t)b * NT;
  const TP* rules = rules_all + (size_t)b * NT * S2;
  const TP* emis = emis_all + (size_t)b * n * PT;
  const TP* sticky = sticky_all ? sticky_all + (size_t)b * n * n : nullptr;
  double* chart = chart_all + (size_t)b * n * n * S;
  int8_t* mask = mask_all + (size_t)b * num * n * n;
  const double* g = kLog ? noise_all + (size_t)b * cap : nullptr;
  auto STK = [&](int i, int j) -> double { return sticky ? (double)sticky[i * n + j] : 0.0; };
  auto CH = [&](int i, int j) -> double* { return chart + ((size_t)i * n + j) * S; };
  if (tid == 0) badsh = 0;
  __syncthreads();
  {
    int bad = 0;
    for (int e = tid; e < NT * S2; e += kThreads) bad |= bad_value(rules[e]);
    for (int e = tid; e < NT; e += kThreads) bad |= bad_value(root[e]);
    for (int e = tid; e < n * PT; e += kThreads) bad |= bad_value(emis[e]);
    if (sticky)
      for (int e = tid; e < n * n; e += kThreads) bad |= !((double)sticky[e] == 0.0 || (double)sticky[e] == ninfd());
    if (bad) atomicOr(&badsh, 1);
    for (int e = tid; e < num * n * n; e += kThreads) mask[e] = 0;
  }
  for (int e = tid; e < n * S; e += kThreads) {
    const int i = e / S, X = e - i * S;
    CH(i, i)[X] = (X >= NT) ? (double)emis[i * PT + X - NT] + STK(i, i) : ninfd();
  }
  __syncthreads();
  for (int w = 2; w <= n; ++w) {
    for (int i = 0; i + w - 1 < n; ++i) {
      const int j = i + w - 1;
      for (int e = tid; e < S2; e += kThreads) {
        const int Bq = e / S, Cq = e - Bq * S;
        double m = ninfd();
        for (int k = i; k < j; ++k) m = fmax(m, CH(i, k)[Bq] + CH(k + 1, j)[Cq]);
        if (kLog && m != ninfd()) {  // logsumexp over the split (constituency.py:262)
          double sm = 0.0;
          for (int k = i; k < j; ++k) sm += exp(CH(i, k)[Bq] + CH(k + 1, j)[Cq] - m);
          m = log(sm) + m;
        }
        pairs[e] = m;
      }
      __syncthreads();
      for (int A = warp; A < S; A += kWarps) {
        double m = ninfd();
        if (A < NT) {
          const TP* ra = rules + (size_t)A * S2;
          if (!kLog) {
            for (int e = lane; e < S2; e += 32) m = fmax(m, (double)ra[e] + pairs[e]);
            m = warp_maxd(m);
          } else {
            // lse over C per B (lanes over B), then over B (constituency.py:263-264); the
            // per-B values are combined with an online (max, sum) so any S works
            double lm = ninfd(), ls = 0.0;
            for (int Bq = lane; Bq < S; Bq += 32) {
              double mx = ninfd();
              for (int Cq = 0; Cq < S; ++Cq) mx = fmax(mx, (double)ra[Bq * S + Cq] + pairs[Bq * S + Cq]);
              if (mx == ninfd()) continue;
              double sm = 0.0;
              for (int Cq = 0; Cq < S; ++Cq) sm += exp((double)ra[Bq * S + Cq] + pairs[Bq * S + Cq] - mx);
              const double vb = log(sm) + mx;
              if (vb > lm) {
                ls = (lm == ninfd() ? 0.0 : ls * exp(lm - vb)) + 1.0;
                lm = vb;
              } else {
                ls += exp(vb - lm);
              }
            }
            double mx = warp_maxd(lm);
            double sm = 0.0;
            if (mx != ninfd()) {
              sm = (lm == ninfd()) ? 0.0 : ls * exp(lm - mx);
              for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
              mx = log(sm) + mx;
            }
            m = mx;
          }
        }
        if (lane == 0) CH(i, j)[A] = (A < NT) ? m + STK(i, j) : ninfd();
      }
      __syncthreads();
    }
  }
  // root pick (constituency.py:346)
  ArgBest x{ninfd(), 1 << 30};
  for (int A = tid; A < NT; A += kThreads) x = arg_better(x, ArgBest{(double)root[A] + CH(0, n - 1)[A], A});
  const ArgBest r0 = block_argmax(x, red);
  const double best = (n == 1) ? ninfd() : r0.v;  // a width-1 sentence has no NT derivation
  if (tid == 0) {
    status[b] = badsh ? SDB_ST_INVALID : (best == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
    if (score) score[b] = best;
    if (used) used[b] = 0;
  }
  if (badsh || best == ninfd()) return;
  int64_t pos = 0;
  for (int rr = 0; rr < num; ++rr) {
  int8_t* maskr = mask + (size_t)rr * n * n;
  ArgBest rp = r0;
  if (kLog) {  // root symbol ~ exp(root + chart[0, n-1]) (constituency.py:346)
    ArgBest y{ninfd(), 1 << 30};
    for (int A = tid; A < NT; A += kThreads) {
      const double w = (double)root[A] + CH(0, n - 1)[A];
      if (w > ninfd()) y = arg_better(y, ArgBest{w + g[pos + A], A});
    }
    rp = block_argmax(y, red);
    pos += NT;
  }
  // walk (stack order is irrelevant for the span mask)
  int top = 0;
  if (tid == 0) {
    stk_i[0] = 0;
    stk_j[0] = n - 1;
    stk_a[0] = rp.i;
  }
  top = 1;
  __syncthreads();
  while (top > 0) {
    --top;
    const int i = stk_i[top], j = stk_j[top], a = stk_a[top];
    __syncthreads();
    if (tid == 0) maskr[i * n + j] = 1;
    if (i == j) continue;
    const int width = j - i;
    const TP* ra = rules + (size_t)a * S2;
    ArgBest y{ninfd(), 1 << 30};
    for (int e = tid; e < width * S2; e += kThreads) {
      const int ko = e / S2, r = e - ko * S2, Bq = r / S, Cq = r - Bq * S;
      const int k = i + ko;
      const double v = ((double)ra[r] + CH(i, k)[Bq]) + CH(k + 1, j)[Cq];
      if (!kLog) {
        if (v > y.v) y = ArgBest{v, e};
      } else if (v > ninfd()) {
        y = arg_better(y, ArgBest{v + g[pos + e], e});
      }
    }
    const ArgBest pk = block_argmax(y, red);
    if (kLog) pos += (int64_t)width * S2;
    const int ko = pk.i / S2, r = pk.i - ko * S2, Bq = r / S, Cq = r - Bq * S;
    const int k = i + ko;
    if (tid == 0) {
      stk_i[top] = i;
      stk_j[top] = k;
      stk_a[top] = Bq;
      stk_i[top + 1] = k + 1;
      stk_j[top + 1] = j;
      stk_a[top + 1] = Cq;
    }
    top += 2;
    __syncthreads();
  }
  }
  if (kLog && tid == 0) used[b] = (int32_t)pos;
}

template <int kMode>
int pcfg_launch(const float* root, const float* rules, const float* emissions, const float* sticky, int64_t B, int n,
                int NT, int PT, PcfgWs ws, double* logz, float* span_marg, PcfgGradOut gout, int32_t* status,
                cudaStream_t s) {
  const size_t smem_in = (size_t)(3 * kBS * 1024 + kMaxN * 3 * kBS * 32 + (kMode == 2 ? kMaxN * 32 : 0)) * 4;
  const size_t smem_out = (size_t)(2 * 3 * kBS * 1024 + kCP * 32 + kCP * 3 * 32 * 33) * 4;
  const size_t smem = kMode == 0 ? smem_in : (smem_in > smem_out ? smem_in : smem_out);
  if (sdb_set_smem((const void*)pcfg_kernel<kMode>, smem) != cudaSuccess)
    return SDB_ERR_CUDA;
  pcfg_kernel<kMode><<<(unsigned)B, kPT, smem, s>>>(root, rules, emissions, sticky, n, NT, PT, ws, logz,
                                                         span_marg, gout, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

int pcfg_check(int64_t B, int n, int NT, int PT) {
  if (B < 0 || n < 1 || NT < 1 || PT < 1) return SDB_ERR_ARG;
  if (n > 1024 || NT + PT > 1024) return SDB_ERR_UNSUPPORTED;
  return SDB_OK;
}

// the register / shared-memory specialised inside-outside kernel; other shapes take pcfg_gen.cu
bool pcfg_fast(int n, int NT, int PT) { return n <= kMaxN && NT <= 32 && PT <= 32; }

size_t max_smem(int n, int NT, int PT) {
  return (size_t)(NT + PT) * (NT + PT) * sizeof(double) + (size_t)6 * n * sizeof(int);
}

}  // namespace

extern "C" size_t sdb_pcfg_fb_workspace(int64_t B, int32_t n, int32_t NT, int32_t PT) {
  if (!pcfg_fast(n, NT, PT)) return pcfg_gen_workspace(B, n, NT, PT, false);
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
  cudaStream_t s = (cudaStream_t)stream;
  if (!pcfg_fast(n, NT, PT))
    return pcfg_gen_launch(span_marg ? 1 : 0, root, rules, emissions, sticky, B, n, NT, PT, logz, span_marg, nullptr,
                           nullptr, nullptr, status, workspace, ws_bytes, s);
  size_t need = 0;
  PcfgWs ws = pcfg_carve(workspace, B, n, NT, PT, &need);
  if (!workspace || ws_bytes < need) return SDB_ERR_WORKSPACE;
  return span_marg ? pcfg_launch<1>(root, rules, emissions, sticky, B, n, NT, PT, ws, logz, span_marg, PcfgGradOut{},
                                    status, s)
                   : pcfg_launch<0>(root, rules, emissions, sticky, B, n, NT, PT, ws, logz, nullptr, PcfgGradOut{},
                                    status, s);
}

extern "C" size_t sdb_pcfg_grad_workspace(int64_t B, int32_t n, int32_t NT, int32_t PT) {
  if (!pcfg_fast(n, NT, PT)) return pcfg_gen_workspace(B, n, NT, PT, true);
  size_t bytes = 0;
  pcfg_carve(nullptr, B, n, NT, PT, &bytes, true);
  return bytes;
}

extern "C" int sdb_pcfg_grad(const float* root, const float* rules, const float* emissions, const float* sticky,
                             int64_t B, int32_t n, int32_t NT, int32_t PT, double* logz, float* span_marg,
                             float* grad_root, float* grad_rules, float* grad_emissions, int32_t* status,
                             void* workspace, size_t ws_bytes, void* stream) {
  int rc = pcfg_check(B, n, NT, PT);
  if (rc) return rc;
  if (!root || !rules || !emissions || !logz || !span_marg || !grad_root || !grad_rules || !grad_emissions || !status)
    return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!pcfg_fast(n, NT, PT))
    return pcfg_gen_launch(2, root, rules, emissions, sticky, B, n, NT, PT, logz, span_marg, grad_root, grad_rules,
                           grad_emissions, status, workspace, ws_bytes, (cudaStream_t)stream);
  size_t need = 0;
  PcfgWs ws = pcfg_carve(workspace, B, n, NT, PT, &need, true);
  if (!workspace || ws_bytes < need) return SDB_ERR_WORKSPACE;
  return pcfg_launch<2>(root, rules, emissions, sticky, B, n, NT, PT, ws, logz, span_marg,
                        PcfgGradOut{grad_root, grad_rules, grad_emissions}, status, (cudaStream_t)stream);
}

extern "C" size_t sdb_pcfg_viterbi_workspace(int64_t B, int32_t n, int32_t NT, int32_t PT) {
  return (size_t)B * n * n * (NT + PT) * sizeof(double);
}

extern "C" int sdb_pcfg_viterbi(const float* root, const float* rules, const float* emissions, const float* sticky,
                                int64_t B, int32_t n, int32_t NT, int32_t PT, int8_t* span_mask, double* score,
                                int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  int rc = pcfg_check(B, n, NT, PT);
  if (rc) return rc;
  if (!root || !rules || !emissions || !span_mask || !score || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!workspace || ws_bytes < sdb_pcfg_viterbi_workspace(B, n, NT, PT)) return SDB_ERR_WORKSPACE;
  const size_t smem = max_smem(n, NT, PT);
  if (smem > 220 * 1024) return SDB_ERR_UNSUPPORTED;
  if (sdb_set_smem((const void*)pcfg_max_kernel<false>, smem) !=
      cudaSuccess)
    return SDB_ERR_CUDA;
  pcfg_max_kernel<false><<<(unsigned)B, kThreads, smem, (cudaStream_t)stream>>>(
      root, rules, emissions, sticky, n, NT, PT, (double*)workspace, span_mask, score, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

// exact mode: the same max-plus chart and walk on float64 grammars (the score is
// _pcfg_best_derivation_score, dist.py:157, exactly)
extern "C" int sdb_pcfg_viterbi_f64(const double* root, const double* rules, const double* emissions,
                                    const double* sticky, int64_t B, int32_t n, int32_t NT, int32_t PT,
                                    int8_t* span_mask, double* score, int32_t* status, void* workspace,
                                    size_t ws_bytes, void* stream) {
  int rc = pcfg_check(B, n, NT, PT);
  if (rc) return rc;
  if (!root || !rules || !emissions || !span_mask || !score || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!workspace || ws_bytes < sdb_pcfg_viterbi_workspace(B, n, NT, PT)) return SDB_ERR_WORKSPACE;
  const size_t smem = max_smem(n, NT, PT);
  if (smem > 220 * 1024) return SDB_ERR_UNSUPPORTED;
  if (sdb_set_smem((const void*)pcfg_max_kernel<false, double>, smem) != cudaSuccess) return SDB_ERR_CUDA;
  pcfg_max_kernel<false, double><<<(unsigned)B, kThreads, smem, (cudaStream_t)stream>>>(
      root, rules, emissions, sticky, n, NT, PT, (double*)workspace, span_mask, score, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

// pcfg_sample (constituency.py:374-378): log-semiring chart + Gumbel-max
// derivation walk over the caller's stream (bound per sample: NT + S^2 n(n-1)/2).
extern "C" int sdb_pcfg_sample(const float* root, const float* rules, const float* emissions, const float* sticky,
                               int64_t B, int32_t n, int32_t NT, int32_t PT, const double* noise,
                               int64_t noise_per_instance, int32_t num, int8_t* span_mask, int32_t* used,
                               int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  int rc = pcfg_check(B, n, NT, PT);
  if (rc) return rc;
  if (!root || !rules || !emissions || !noise || !span_mask || !used || !status || num < 1) return SDB_ERR_ARG;
  const int64_t S = NT + PT;
  if (noise_per_instance < (int64_t)num * (NT + S * S * ((int64_t)n * (n - 1) / 2))) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!workspace || ws_bytes < sdb_pcfg_viterbi_workspace(B, n, NT, PT)) return SDB_ERR_WORKSPACE;
  const size_t smem = max_smem(n, NT, PT);
  if (smem > 220 * 1024) return SDB_ERR_UNSUPPORTED;
  if (sdb_set_smem((const void*)pcfg_max_kernel<true>, smem) !=
      cudaSuccess)
    return SDB_ERR_CUDA;
  pcfg_max_kernel<true><<<(unsigned)B, kThreads, smem, (cudaStream_t)stream>>>(
      root, rules, emissions, sticky, n, NT, PT, (double*)workspace, span_mask, nullptr, status, noise,
      noise_per_instance, num, used);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
