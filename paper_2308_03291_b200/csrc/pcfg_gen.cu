// PCFG inside / outside for grammars and sentences outside the fast kernel's
// shape (pcfg.cu: n <= 64, NT <= 32, PT <= 32) -- e.g. the paper's benchmark
// grammar NT=64, PT=96.
//
// Reference: structdist constituency.py:246-340 (_pcfg_inside, pcfg_inside,
// pcfg_gradients).  Same layouts as pcfg.cu.
//
// One CTA (512 threads) per instance; fp64 scaled-LINEAR charts: every span
// (i,j) holds u_ij[X] = exp(chart[i,j,X] - s_ij) over all S = NT+PT symbols
// with an fp64 log scale s_ij (-inf = empty).  Positive sums only, so the
// result is exact to fp64 rounding.  Per span of width w (widths ascending):
//   pair  P[B][C] = sum_k exp(s_ik + s_(k+1)j - m) u_ik[B] u_(k+1)j[C]
//   inner[A] = sum_{B,C} exp(rules[A,B,C]) P[B][C]            (NT x S^2)
// Outside, parents by width descending (push form, constituency.py:303-325):
//   Q[B][C] = sum_A o_p[A] exp(rules[A,B,C]);  left child  += Q u_right,
//   right child += Q^T u_left, accumulated with scaled (vector, log scale)
//   adds; rule counts G[A][B][C] += o_p[A] P_p[B][C] (P_p recomputed).
// The big arrays (exp(rules), charts, P, Q, G) live in the workspace (L2
// resident); the kernel is FP64-FMA bound: ~(3 NT + 3 w) S^2 per span.
#include "common.cuh"

namespace {

constexpr int kGT = 512;
constexpr int kGW = kGT / 32;

struct GenWs {
  double* Rl;  // [B][NT][S*S] exp(rules)
  double* iu;  // [B][n][n][S]
  double* is;  // [B][n][n]
  double* ou;  // [B][n][n][S]
  double* os;  // [B][n][n]
  double* P;   // [B][S*S]
  double* Q;   // [B][S*S]
  double* G;   // [B][NT][S*S] (gradients only)
};

GenWs gen_carve(void* base, int64_t B, int n, int NT, int PT, bool grad, size_t* bytes) {
  const size_t S = (size_t)NT + PT, S2 = S * S;
  Carve c(base);
  GenWs w;
  w.Rl = c.take<double>((size_t)B * NT * S2);
  w.iu = c.take<double>((size_t)B * n * n * S);
  w.is = c.take<double>((size_t)B * n * n);
  w.ou = c.take<double>((size_t)B * n * n * S);
  w.os = c.take<double>((size_t)B * n * n);
  w.P = c.take<double>((size_t)B * S2);
  w.Q = c.take<double>((size_t)B * S2);
  w.G = grad ? c.take<double>((size_t)B * NT * S2) : nullptr;
  *bytes = c.used;
  return w;
}

__device__ double block_max_d(double v, double* red) {
  v = warp_maxd(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = red[0];
  for (int i = 1; i < kGW; ++i) r = fmax(r, red[i]);
  return r;
}

__device__ double block_sum_d(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  for (int i = 0; i < kGW; ++i) r += red[i];
  return r;
}

// pair products of span (i, j) into P; returns the common log scale m (-inf: no split)
__device__ double build_pairs(const double* iu, const double* is, int n, int S, int i, int j, double* P,
                              double* red) {
  double m = ninfd();
  for (int k = i; k < j; ++k) m = fmax(m, is[i * n + k] + is[(k + 1) * n + j]);
  if (m == ninfd()) return m;
  const int S2 = S * S;
  for (int e = threadIdx.x; e < S2; e += kGT) {
    const int Bq = e / S, Cq = e - Bq * S;
    double acc = 0.0;
    for (int k = i; k < j; ++k) {
      const double f = is[i * n + k] + is[(k + 1) * n + j] - m;
      if (f == ninfd()) continue;
      acc = fma(exp(f) * iu[((size_t)i * n + k) * S + Bq], iu[((size_t)(k + 1) * n + j) * S + Cq], acc);
    }
    P[e] = acc;
  }
  (void)red;
  return m;
}

// kMode: 0 log Z, 1 + span marginals, 2 + root / rule / emission gradients
template <int kMode, typename TP, typename M>  // TP / M: input / output types (float64 = exact mode)
__global__ void __launch_bounds__(kGT) pcfg_gen_kernel(
    const TP* __restrict__ root_all, const TP* __restrict__ rules_all, const TP* __restrict__ emis_all,
    const TP* __restrict__ sticky_all, int n, int NT, int PT, GenWs ws, double* __restrict__ logz,
    M* __restrict__ marg_all, M* __restrict__ groot_all, M* __restrict__ grules_all,
    M* __restrict__ gemis_all, int32_t* __restrict__ status) {
  __shared__ double red[kGW];
  __shared__ int badsh;
  const int S = NT + PT, S2 = S * S;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const TP* root = root_all + (size_t)b * NT;
  const TP* rules = rules_all + (size_t)b * NT * S2;
  const TP* emis = emis_all + (size_t)b * n * PT;
  const TP* sticky = sticky_all ? sticky_all + (size_t)b * n * n : nullptr;
  double* Rl = ws.Rl + (size_t)b * NT * S2;
  double* iu = ws.iu + (size_t)b * n * n * S;
  double* is = ws.is + (size_t)b * n * n;
  double* ou = ws.ou + (size_t)b * n * n * S;
  double* os = ws.os + (size_t)b * n * n;
  double* P = ws.P + (size_t)b * S2;
  double* Q = ws.Q + (size_t)b * S2;
  double* G = kMode == 2 ? ws.G + (size_t)b * NT * S2 : nullptr;
  auto STK = [&](int i, int j) -> double { return sticky ? (double)sticky[i * n + j] : 0.0; };
  if (tid == 0) badsh = 0;
  __syncthreads();
  {
    int bad = 0;
    for (int e = tid; e < NT * S2; e += kGT) {
      const TP r = rules[e];
      bad |= bad_value(r);
      Rl[e] = exp((double)r);
      if (kMode == 2) G[e] = 0.0;
    }
    for (int e = tid; e < NT; e += kGT) bad |= bad_value(root[e]);
    for (int e = tid; e < n * PT; e += kGT) bad |= bad_value(emis[e]);
    if (sticky)
      for (int e = tid; e < n * n; e += kGT) bad |= !((double)sticky[e] == 0.0 || (double)sticky[e] == ninfd());
    if (bad) atomicOr(&badsh, 1);
  }
  // ---- inside, width 1: preterminal slots = emissions + sticky (constituency.py:255-256)
  for (int i = 0; i < n; ++i) {
    double mx = ninfd();
    for (int X = tid; X < PT; X += kGT) mx = fmax(mx, (double)emis[i * PT + X] + STK(i, i));
    mx = block_max_d(mx, red);
    for (int X = tid; X < S; X += kGT) {
      const double v = X >= NT ? (double)emis[i * PT + X - NT] + STK(i, i) : ninfd();
      iu[((size_t)i * n + i) * S + X] = (mx == ninfd() || v == ninfd()) ? 0.0 : exp(v - mx);
    }
    if (tid == 0) is[i * n + i] = mx;
  }
  __syncthreads();
  // ---- inside, wider spans (constituency.py:257-265)
  for (int w = 2; w <= n; ++w) {
    for (int i = 0; i + w - 1 < n; ++i) {
      const int j = i + w - 1;
      const double m = build_pairs(iu, is, n, S, i, j, P, red);
      __syncthreads();
      double* u = iu + ((size_t)i * n + j) * S;
      double lmax = ninfd();
      if (m != ninfd() && STK(i, j) != ninfd()) {
        for (int A = warp; A < NT; A += kGW) {
          const double* ra = Rl + (size_t)A * S2;
          double acc = 0.0;
          for (int e = lane; e < S2; e += 32) acc = fma(ra[e], P[e], acc);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          if (lane == 0) u[A] = acc;
          lmax = fmax(lmax, acc);
        }
      }
      for (int X = NT + tid; X < S; X += kGT) u[X] = 0.0;
      const double Mx = block_max_d(lane == 0 ? lmax : ninfd(), red);  // (includes the barrier)
      const bool live = Mx > 0.0 && Mx != ninfd();
      for (int A = tid; A < NT; A += kGT) u[A] = live ? u[A] / Mx : 0.0;
      if (tid == 0) is[i * n + j] = live ? m + log(Mx) + STK(i, j) : ninfd();
      __syncthreads();
    }
  }
  // ---- log Z = lse_A root[A] + chart[0, n-1, A]
  double z;
  {
    const double* u = iu + (size_t)(n - 1) * S;
    const double s0 = is[n - 1];
    double mx = ninfd();
    for (int A = tid; A < NT; A += kGT) mx = fmax(mx, (double)root[A]);
    mx = block_max_d(mx, red);
    double acc = 0.0;
    if (n > 1 && s0 != ninfd() && mx != ninfd())
      for (int A = tid; A < NT; A += kGT) acc += exp((double)root[A] - mx) * u[A];
    acc = block_sum_d(acc, red);
    z = (acc > 0.0) ? s0 + mx + log(acc) : ninfd();
    if (tid == 0) {
      logz[b] = badsh ? ninfd() : z;
      status[b] = badsh ? SDB_ST_INVALID : (z == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
    }
  }
  if (kMode == 0) return;
  const bool ok = !badsh && z != ninfd();
  M* marg = marg_all + (size_t)b * n * n;
  if (!ok) {
    for (int e = tid; e < n * n; e += kGT) marg[e] = 0.f;
    if (kMode == 2) {
      for (int e = tid; e < NT; e += kGT) groot_all[(size_t)b * NT + e] = 0.f;
      for (int e = tid; e < NT * S2; e += kGT) grules_all[(size_t)b * NT * S2 + e] = 0.f;
      for (int e = tid; e < n * PT; e += kGT) gemis_all[(size_t)b * n * PT + e] = 0.f;
    }
    return;
  }
  // ---- outside: root span (outside[0, n-1, :NT] = root), everything else empty
  for (int e = tid; e < n * n; e += kGT) os[e] = ninfd();
  __syncthreads();
  {
    double mx = ninfd();
    for (int A = tid; A < NT; A += kGT) mx = fmax(mx, (double)root[A]);
    mx = block_max_d(mx, red);
    double* o = ou + (size_t)(n - 1) * S;
    for (int X = tid; X < S; X += kGT) o[X] = (X < NT && mx != ninfd()) ? exp((double)root[X] - mx) : 0.0;
    if (tid == 0) os[n - 1] = mx;
  }
  __syncthreads();
  // scaled accumulate of (v[S], tau) into child c
  auto accumulate = [&](int c, double tau, const double* v) {
    double* o = ou + (size_t)c * S;
    const double t = os[c];
    const double mm = fmax(t, tau);
    const double fa = (t == ninfd()) ? 0.0 : exp(t - mm);
    const double fb = exp(tau - mm);
    for (int X = tid; X < S; X += kGT) o[X] = (t == ninfd() ? 0.0 : o[X] * fa) + v[X] * fb;
    __syncthreads();
    if (tid == 0) os[c] = mm;
    __syncthreads();
  };
  for (int w = n; w >= 2; --w) {
    for (int i = 0; i + w - 1 < n; ++i) {
      const int j = i + w - 1;
      const double tp = os[i * n + j] + STK(i, j);  // out_span = outside + sticky (constituency.py:306)
      if (tp == ninfd()) continue;
      const double* op = ou + ((size_t)i * n + j) * S;
      // Q[B][C] = sum_A o_p[A] exp(rules[A,B,C])
      for (int e = tid; e < S2; e += kGT) {
        double acc = 0.0;
        for (int A = 0; A < NT; ++A) acc = fma(op[A], Rl[(size_t)A * S2 + e], acc);
        Q[e] = acc;
      }
      double mp = ninfd();
      if (kMode == 2) mp = build_pairs(iu, is, n, S, i, j, P, red);
      __syncthreads();
      if (kMode == 2 && mp != ninfd()) {  // expected rule counts, before the exp(rule) factor
        const double cf = exp(tp + mp - z);
        for (int e = tid; e < NT * S2; e += kGT) {
          const int A = e / S2, r = e - A * S2;
          G[e] = fma(cf * op[A], P[r], G[e]);
        }
      }
      __syncthreads();
      // pushes (constituency.py:318-325); the child vectors are built in the P buffer
      double* v = P;
      for (int k = i; k < j; ++k) {
        const double sr = is[(k + 1) * n + j], sl = is[i * n + k];
        if (sr != ninfd()) {  // left child (i,k) += Q u_right
          const double* ur = iu + ((size_t)(k + 1) * n + j) * S;
          for (int Bq = tid; Bq < S; Bq += kGT) {
            double acc = 0.0;
            for (int Cq = 0; Cq < S; ++Cq) acc = fma(Q[Bq * S + Cq], ur[Cq], acc);
            v[Bq] = acc;
          }
          __syncthreads();
          accumulate(i * n + k, tp + sr, v);
        }
        if (sl != ninfd()) {  // right child (k+1,j) += Q^T u_left
          const double* ul = iu + ((size_t)i * n + k) * S;
          for (int Cq = tid; Cq < S; Cq += kGT) {
            double acc = 0.0;
            for (int Bq = 0; Bq < S; ++Bq) acc = fma(Q[Bq * S + Cq], ul[Bq], acc);
            v[Cq] = acc;
          }
          __syncthreads();
          accumulate((k + 1) * n + j, tp + sl, v);
        }
      }
    }
  }
  // ---- span marginals: exp(lse(outside + chart) - Z) (constituency.py:330-334)
  for (int c = warp; c < n * n; c += kGW) {
    const int i = c / n, j = c - i * n;
    double val = 0.0;
    if (j >= i) {
      const double t = os[c], s = is[c];
      double acc = 0.0;
      if (t != ninfd() && s != ninfd())
        for (int X = lane; X < S; X += 32) acc = fma(ou[(size_t)c * S + X], iu[(size_t)c * S + X], acc);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (acc > 0.0) val = exp(log(acc) + t + s - z);
    }
    if (lane == 0) marg[c] = (M)val;
  }
  if (kMode != 2) return;
  // ---- gradients (constituency.py:326-329)
  {
    const double* u = iu + (size_t)(n - 1) * S;
    const double s0 = is[n - 1];
    for (int A = tid; A < NT; A += kGT)
      groot_all[(size_t)b * NT + A] =
          (M)((s0 == ninfd() || u[A] == 0.0) ? 0.0 : exp((double)root[A] + s0 + log(u[A]) - z));
    for (int e = tid; e < NT * S2; e += kGT) grules_all[(size_t)b * NT * S2 + e] = (M)(G[e] * Rl[e]);
    for (int e = tid; e < n * PT; e += kGT) {
      const int i = e / PT, X = e - i * PT;
      const double t = os[i * n + i];
      const double o = ou[((size_t)i * n + i) * S + NT + X];
      const double v = (t == ninfd() || o == 0.0) ? ninfd() : log(o) + t + STK(i, i) + (double)emis[e] - z;
      gemis_all[(size_t)b * n * PT + e] = (M)(v == ninfd() ? 0.0 : exp(v));
    }
  }
}

}  // namespace

size_t pcfg_gen_workspace(int64_t B, int n, int NT, int PT, bool grad) {
  size_t bytes = 0;
  gen_carve(nullptr, B, n, NT, PT, grad, &bytes);
  return bytes;
}

template <typename TP, typename M>
int pcfg_gen_launch_t(int mode, const TP* root, const TP* rules, const TP* emissions, const TP* sticky, int64_t B,
                      int n, int NT, int PT, double* logz, M* span_marg, M* groot, M* grules, M* gemis,
                      int32_t* status, void* workspace, size_t ws_bytes, cudaStream_t s) {
  size_t need = 0;
  GenWs ws = gen_carve(workspace, B, n, NT, PT, mode == 2, &need);
  if (!workspace || ws_bytes < need) return SDB_ERR_WORKSPACE;
  if (mode == 0)
    pcfg_gen_kernel<0, TP, M><<<(unsigned)B, kGT, 0, s>>>(root, rules, emissions, sticky, n, NT, PT, ws, logz,
                                                           nullptr, nullptr, nullptr, nullptr, status);
  else if (mode == 1)
    pcfg_gen_kernel<1, TP, M><<<(unsigned)B, kGT, 0, s>>>(root, rules, emissions, sticky, n, NT, PT, ws, logz,
                                                           span_marg, nullptr, nullptr, nullptr, status);
  else
    pcfg_gen_kernel<2, TP, M><<<(unsigned)B, kGT, 0, s>>>(root, rules, emissions, sticky, n, NT, PT, ws, logz,
                                                           span_marg, groot, grules, gemis, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

int pcfg_gen_launch(int mode, const float* root, const float* rules, const float* emissions, const float* sticky,
                    int64_t B, int n, int NT, int PT, double* logz, float* span_marg, float* groot, float* grules,
                    float* gemis, int32_t* status, void* workspace, size_t ws_bytes, cudaStream_t s) {
  return pcfg_gen_launch_t<float, float>(mode, root, rules, emissions, sticky, B, n, NT, PT, logz, span_marg, groot,
                                         grules, gemis, status, workspace, ws_bytes, s);
}

// ---- exact mode (float64 grammar / emissions / sticky in, float64 span marginals and gradients out)
extern "C" size_t sdb_pcfg_f64_workspace(int64_t B, int32_t n, int32_t NT, int32_t PT, int32_t grad) {
  return (B < 0 || n < 1 || NT < 1 || PT < 1) ? 0 : pcfg_gen_workspace(B, n, NT, PT, grad != 0);
}
// span_marg == NULL: log Z only; groot/grules/gemis non-NULL (with span_marg): the gradients too
extern "C" int sdb_pcfg_f64(const double* root, const double* rules, const double* emissions, const double* sticky,
                            int64_t B, int32_t n, int32_t NT, int32_t PT, double* logz, double* span_marg,
                            double* groot, double* grules, double* gemis, int32_t* status, void* workspace,
                            size_t ws_bytes, void* stream) {
  if (B < 0 || n < 1 || NT < 1 || PT < 1 || !root || !rules || !emissions || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  const int mode = !span_marg ? 0 : (groot && grules && gemis) ? 2 : 1;
  return pcfg_gen_launch_t<double, double>(mode, root, rules, emissions, sticky, B, n, NT, PT, logz, span_marg, groot,
                                           grules, gemis, status, workspace, ws_bytes, (cudaStream_t)stream);
}
