// Exact sampling (forward filtering, backward sampling with Gumbel-max
// picks) and the Eisner max-plus decode.
//
// Reference: dist.py:179-212 (sample_info: ONE numpy Generator stream per
// call, num samples drawn back to back), numerics.py:162-168
// (sample_log_categorical: g = rng.gumbel(size=len(w)); argmax(where(w > -inf,
// w + g, -inf)), first maximum), chain.py:117-129, alignment.py:121-150,
// 304-343, constituency.py:113-140, spanning.py:283-331.
//
// The Gumbel stream is drawn on the host by the caller from the same
// Generator (numpy draws element by element, so one long gumbel(size=N) call
// equals the reference's per-pick calls) and consumed here in the
// reference's pick order; every kernel reports how many draws it used.  The
// charts are fp64 in the log semiring with the reference's max-shifted
// log-sum-exp, so the picks match the reference's (the walks are sequential
// and tiny; the charts are the parallel part).
//
// One CTA per instance: the chart is built by all threads, then thread 0 (or
// the block, for the chain's m-way picks) walks num samples.
#include "common.cuh"

namespace {

constexpr int kT = 256;

__device__ __forceinline__ double lse2(double m, double s) { return m == ninfd() ? ninfd() : log(s) + m; }

// first maximum of w + g over the entries with w > -inf (numerics.py:167-168)
struct Pick {
  double best;
  int idx;
};
__device__ __forceinline__ void pick_add(Pick& p, double w, double g, int k) {
  if (w > ninfd()) {
    const double v = w + g;
    if (p.idx < 0 || v > p.best) {
      p.best = v;
      p.idx = k;
    }
  }
}

// ================================================================ chain
// chain.py:64-70 (alpha) and 117-129 (FFBS).  Thread per tag.
__global__ void __launch_bounds__(1024) chain_sample_kernel(const float* __restrict__ init_all,
                                                             const float* __restrict__ trans_all, int n, int m,
                                                             const double* __restrict__ noise_all, int64_t cap,
                                                             int num, double* __restrict__ al_all,
                                                             int32_t* __restrict__ tags_all, int32_t* __restrict__ used,
                                                             int32_t* __restrict__ status) {
  __shared__ double rv[32];
  __shared__ int ri[32];
  __shared__ int tag_s;
  const int b = blockIdx.x, y = threadIdx.x, lane = y & 31, warp = y >> 5, nw = (blockDim.x + 31) >> 5;
  const float* init = init_all + (size_t)b * m;
  const float* tr = trans_all + (size_t)b * (n - 1) * m * m;
  double* al = al_all + (size_t)b * n * m;
  const double* g = noise_all + (size_t)b * cap;
  int bad = 0;
  if (y < m) {
    al[y] = (double)init[y];
    bad |= bad_input(init[y]);
  }
  __syncthreads();
  for (int t = 0; t + 1 < n; ++t) {
    if (y < m) {
      const float* tt = tr + (size_t)t * m * m;
      double mx = ninfd();
      for (int x = 0; x < m; ++x) {
        bad |= bad_input(tt[x * m + y]);
        mx = fmax(mx, al[(size_t)t * m + x] + (double)tt[x * m + y]);
      }
      double s = 0.0;
      if (mx != ninfd())
        for (int x = 0; x < m; ++x) s += exp(al[(size_t)t * m + x] + (double)tt[x * m + y] - mx);
      al[(size_t)(t + 1) * m + y] = lse2(mx, s);
    }
    __syncthreads();
  }
  const int anybad = __syncthreads_or(bad);
  const int alive = __syncthreads_or(y < m && al[(size_t)(n - 1) * m + y] > ninfd());
  if (y == 0) status[b] = anybad ? SDB_ST_INVALID : (alive ? SDB_ST_OK : SDB_ST_VACUOUS);
  if (anybad || !alive) {
    if (y == 0) used[b] = 0;
    return;
  }
  int64_t pos = 0;
  for (int r = 0; r < num; ++r) {
    int32_t* tags = tags_all + ((size_t)b * num + r) * n;
    int next = -1;
    for (int t = n - 1; t >= 0; --t) {
      Pick p{ninfd(), -1};
      if (y < m) {
        const double w = al[(size_t)t * m + y] +
                         (t == n - 1 ? 0.0 : (double)tr[((size_t)t * m + y) * m + next]);
        pick_add(p, w, g[pos + y], y);
      }
      // block first-max
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, p.best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, p.idx, o);
        if (oi >= 0 && (p.idx < 0 || ov > p.best || (ov == p.best && oi < p.idx))) {
          p.best = ov;
          p.idx = oi;
        }
      }
      if (lane == 0) {
        rv[warp] = p.best;
        ri[warp] = p.idx;
      }
      __syncthreads();
      if (y == 0) {
        Pick q{ninfd(), -1};
        for (int x = 0; x < nw; ++x)
          if (ri[x] >= 0 && (q.idx < 0 || rv[x] > q.best || (rv[x] == q.best && ri[x] < q.idx))) q = Pick{rv[x], ri[x]};
        tag_s = q.idx;
        tags[t] = q.idx;
      }
      __syncthreads();
      next = tag_s;
      pos += m;
    }
  }
  if (y == 0) used[b] = (int32_t)pos;
}

// ============================================================ alignment
// alignment.py:62-77 (alpha, lse over the in-grid sources in DIAG, DOWN,
// RIGHT order) and 121-150 (walk from (n, m)).
__global__ void __launch_bounds__(kT) nw_sample_kernel(const float* __restrict__ th_all, int n, int m,
                                                       const double* __restrict__ noise_all, int64_t cap, int num,
                                                       double* __restrict__ al_all, int8_t* __restrict__ path_all,
                                                       int32_t* __restrict__ used, int32_t* __restrict__ status) {
  const int b = blockIdx.x, tid = threadIdx.x;
  const int m1 = m + 1;
  const float* th = th_all + (size_t)b * (n + 1) * m1 * 3;
  double* al = al_all + (size_t)b * (n + 1) * m1;
  const double* g = noise_all + (size_t)b * cap;
  int bad = 0;
  if (tid == 0) al[0] = 0.0;
  for (int e = tid; e < 3; e += kT) bad |= bad_input(th[e]);
  __syncthreads();
  for (int d = 1; d <= n + m; ++d) {
    const int i0 = max(0, d - m), i1 = min(n, d);
    for (int i = i0 + tid; i <= i1; i += kT) {
      const int j = d - i;
      const float* c = th + ((size_t)i * m1 + j) * 3;
      double t[3];
      int c3 = 0;
      bad |= bad_input(c[0]) | bad_input(c[1]) | bad_input(c[2]);
      if (i >= 1 && j >= 1) t[c3++] = al[(size_t)(i - 1) * m1 + j - 1] + (double)c[0];
      if (i >= 1) t[c3++] = al[(size_t)(i - 1) * m1 + j] + (double)c[1];
      if (j >= 1) t[c3++] = al[(size_t)i * m1 + j - 1] + (double)c[2];
      double mx = ninfd();
      for (int q = 0; q < c3; ++q) mx = fmax(mx, t[q]);
      double s = 0.0;
      if (mx != ninfd())
        for (int q = 0; q < c3; ++q) s += exp(t[q] - mx);
      al[(size_t)i * m1 + j] = lse2(mx, s);
    }
    __syncthreads();
  }
  const int anybad = __syncthreads_or(bad);
  const bool alive = al[(size_t)n * m1 + m] > ninfd();
  for (int e = tid; e < num * (n + 1) * m1; e += kT) path_all[(size_t)b * num * (n + 1) * m1 + e] = -1;
  __syncthreads();
  if (tid != 0) return;
  status[b] = anybad ? SDB_ST_INVALID : (alive ? SDB_ST_OK : SDB_ST_VACUOUS);
  int64_t pos = 0;
  if (!anybad && alive) {
    for (int r = 0; r < num; ++r) {
      int8_t* path = path_all + ((size_t)b * num + r) * (n + 1) * m1;
      int i = n, j = m;
      while (i != 0 || j != 0) {
        const float* c = th + ((size_t)i * m1 + j) * 3;
        Pick p{ninfd(), -1};
        int k = 0;
        if (i >= 1 && j >= 1) pick_add(p, al[(size_t)(i - 1) * m1 + j - 1] + (double)c[0], g[pos + k++], 0);
        if (i >= 1) pick_add(p, al[(size_t)(i - 1) * m1 + j] + (double)c[1], g[pos + k++], 1);
        if (j >= 1) pick_add(p, al[(size_t)i * m1 + j - 1] + (double)c[2], g[pos + k++], 2);
        pos += k;
        path[(size_t)i * m1 + j] = (int8_t)p.idx;
        if (p.idx == 0) { --i; --j; } else if (p.idx == 1) { --i; } else { --j; }
      }
    }
  }
  used[b] = (int32_t)pos;
}

// ================================================================== CTC
// alignment.py:231-264 (expanded lattice, alpha) and 304-343 (walk).
__global__ void __launch_bounds__(kT) ctc_sample_kernel(const float* __restrict__ fp_all,
                                                        const int32_t* __restrict__ tg_all, int T, int V, int L,
                                                        const double* __restrict__ noise_all, int64_t cap, int num,
                                                        double* __restrict__ al_all, int32_t* __restrict__ st_all,
                                                        int32_t* __restrict__ used, int32_t* __restrict__ status) {
  const int b = blockIdx.x, tid = threadIdx.x;
  const int S = 2 * L + 1;
  const float* fp = fp_all + (size_t)b * T * V;
  const int32_t* tg = tg_all + (size_t)b * L;
  double* al = al_all + (size_t)b * T * S;
  const double* g = noise_all + (size_t)b * cap;
  auto lab = [&](int s) { return (s & 1) ? tg[s >> 1] : 0; };
  auto skip = [&](int s) { return s >= 2 && lab(s) != 0 && lab(s) != lab(s - 2); };
  int bad = 0;
  for (int e = tid; e < T * V; e += kT) bad |= bad_input(fp[e]);
  for (int e = tid; e < L; e += kT) bad |= (tg[e] < 1 || tg[e] >= V);
  const int anybad = __syncthreads_or(bad);
  if (anybad) {
    if (tid == 0) {
      status[b] = SDB_ST_INVALID;
      used[b] = 0;
    }
    return;
  }
  for (int s = tid; s < S; s += kT) al[s] = (s <= 1) ? (double)fp[lab(s)] : ninfd();
  __syncthreads();
  for (int t = 1; t < T; ++t) {
    for (int s = tid; s < S; s += kT) {
      const double* p = al + (size_t)(t - 1) * S;
      double x[3];
      int c = 0;
      x[c++] = p[s];
      if (s >= 1) x[c++] = p[s - 1];
      if (skip(s)) x[c++] = p[s - 2];
      double mx = ninfd();
      for (int q = 0; q < c; ++q) mx = fmax(mx, x[q]);
      double sm = 0.0;
      if (mx != ninfd())
        for (int q = 0; q < c; ++q) sm += exp(x[q] - mx);
      al[(size_t)t * S + s] = lse2(mx, sm) + (double)fp[(size_t)t * V + lab(s)];
    }
    __syncthreads();
  }
  if (tid != 0) return;
  const double* last = al + (size_t)(T - 1) * S;
  const bool alive = last[S - 1] > ninfd() || (S > 1 && last[S - 2] > ninfd());
  status[b] = alive ? SDB_ST_OK : SDB_ST_VACUOUS;
  int64_t pos = 0;
  if (alive) {
    for (int r = 0; r < num; ++r) {
      int32_t* states = st_all + ((size_t)b * num + r) * T;
      Pick p{ninfd(), -1};
      pick_add(p, last[S - 1], g[pos], S - 1);
      if (S > 1) pick_add(p, last[S - 2], g[pos + 1], S - 2);
      pos += (S > 1) ? 2 : 1;
      int s = p.idx;
      states[T - 1] = s;
      for (int t = T - 1; t >= 1; --t) {
        const double* pr = al + (size_t)(t - 1) * S;
        Pick q{ninfd(), -1};
        int k = 0;
        pick_add(q, pr[s], g[pos + k++], s);
        if (s >= 1) pick_add(q, pr[s - 1], g[pos + k++], s - 1);
        if (skip(s)) pick_add(q, pr[s - 2], g[pos + k++], s - 2);
        pos += k;
        s = q.idx;
        states[t - 1] = s;
      }
    }
  }
  used[b] = (int32_t)pos;
}

// ============================================================= Tree-CRF
// constituency.py:52-64 (label fold + inside, lse) and 113-140 (walk, LIFO
// stack: the right child is expanded first).
__global__ void __launch_bounds__(kT) tree_sample_kernel(const float* __restrict__ th_all, int n, int m,
                                                         const double* __restrict__ noise_all, int64_t cap, int num,
                                                         double* __restrict__ ch_all, int32_t* __restrict__ lab_all,
                                                         int32_t* __restrict__ used, int32_t* __restrict__ status) {
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* th = th_all + (size_t)b * n * n * m;
  double* ins = ch_all + (size_t)b * n * n;
  const double* g = noise_all + (size_t)b * cap;
  int bad = 0;
  for (int e = tid; e < n * n * m; e += kT) {
    const int i = e / (n * m), j = (e / m) % n;
    if (i <= j) bad |= bad_input(th[e]);
  }
  const int anybad = __syncthreads_or(bad);
  if (anybad) {
    if (tid == 0) {
      status[b] = SDB_ST_INVALID;
      used[b] = 0;
    }
    return;
  }
  // inside[i][j] = fold[i][j] + lse_k(inside[i][k] + inside[k+1][j]); fold = lse over labels
  for (int w = 1; w <= n; ++w) {
    for (int i = warp; i + w - 1 < n; i += kT / 32) {
      const int j = i + w - 1;
      const float* c = th + ((size_t)i * n + j) * m;
      double mx = ninfd();
      for (int l = lane; l < m; l += 32) mx = fmax(mx, (double)c[l]);
      mx = warp_maxd(mx);
      double s = 0.0;
      if (mx != ninfd())
        for (int l = lane; l < m; l += 32) s += exp((double)c[l] - mx);
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      const double fold = lse2(mx, s);
      double v = fold;
      if (w > 1) {
        double pm = ninfd();
        for (int k = i + lane; k < j; k += 32) pm = fmax(pm, ins[i * n + k] + ins[(k + 1) * n + j]);
        pm = warp_maxd(pm);
        double ps = 0.0;
        if (pm != ninfd())
          for (int k = i + lane; k < j; k += 32) ps += exp(ins[i * n + k] + ins[(k + 1) * n + j] - pm);
        for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
        v = fold + lse2(pm, ps);
      }
      if (lane == 0) ins[i * n + j] = v;
    }
    __syncthreads();
  }
  for (int e = tid; e < num * n * n; e += kT) lab_all[(size_t)b * num * n * n + e] = -1;
  __syncthreads();
  if (tid != 0) return;
  const bool alive = ins[n - 1] > ninfd();
  status[b] = alive ? SDB_ST_OK : SDB_ST_VACUOUS;
  int64_t pos = 0;
  extern __shared__ int tstk[];  // walk stack [2][2n] (dynamic), thread 0 only
  int* si = tstk;
  int* sj = tstk + 2 * n;
  if (alive) {
    for (int r = 0; r < num; ++r) {
      int32_t* lab = lab_all + ((size_t)b * num + r) * n * n;
      int top = 0;
      si[top] = 0;
      sj[top++] = n - 1;
      while (top > 0) {
        --top;
        const int i = si[top], j = sj[top];
        const float* c = th + ((size_t)i * n + j) * m;
        Pick p{ninfd(), -1};
        for (int l = 0; l < m; ++l) pick_add(p, (double)c[l], g[pos + l], l);
        pos += m;
        lab[i * n + j] = p.idx;
        if (i == j) continue;
        Pick q{ninfd(), -1};
        for (int o = 0; o < j - i; ++o) pick_add(q, ins[i * n + i + o] + ins[(i + o + 1) * n + j], g[pos + o], o);
        pos += j - i;
        const int k = i + q.idx;
        si[top] = i;
        sj[top++] = k;
        si[top] = k + 1;
        sj[top++] = j;
      }
    }
  }
  used[b] = (int32_t)pos;
}

// =============================================================== Eisner
// spanning.py:183-207 (charts) and 283-331 (decode; kMax -> max-plus charts
// and first-argmax picks, i.e. eisner_max_arcs).  Charts [4][N][N] fp64:
// cr, cl, ir, il.
template <bool kMax>
__global__ void __launch_bounds__(kT) eisner_decode_kernel(const float* __restrict__ adj_all, int n, int single,
                                                           const double* __restrict__ noise_all, int64_t cap,
                                                           int num, double* __restrict__ ch_all,
                                                           int32_t* __restrict__ heads_all,
                                                           int32_t* __restrict__ used, int32_t* __restrict__ status) {
  const int b = blockIdx.x, tid = threadIdx.x;
  const int N = n + 1;
  const float* th = adj_all + (size_t)b * N * N;
  double* cr = ch_all + (size_t)b * 4 * N * N;
  double* cl = cr + N * N;
  double* ir = cl + N * N;
  double* il = ir + N * N;
  const double* g = kMax ? nullptr : noise_all + (size_t)b * cap;
  int bad = 0;
  for (int e = tid; e < N * N; e += kT) {
    const int h = e / N, d = e - h * N;
    bad |= (h != d && d != 0) ? bad_input(th[e]) : 0;
    cr[e] = cl[e] = ir[e] = il[e] = (h == d) ? 0.0 : ninfd();
  }
  const int anybad = __syncthreads_or(bad);
  if (anybad) {
    if (tid == 0) {
      status[b] = SDB_ST_INVALID;
      used[b] = 0;
    }
    return;
  }
  for (int e = tid; e < N; e += kT) ir[e * N + e] = il[e * N + e] = ninfd();
  __syncthreads();
  // reduce over a strided sequence: max (kMax) or max-shifted log-sum-exp
  auto red = [&](auto f, int cnt) -> double {
    double mx = ninfd();
    for (int q = 0; q < cnt; ++q) mx = fmax(mx, f(q));
    if (kMax || mx == ninfd()) return mx;
    double s = 0.0;
    for (int q = 0; q < cnt; ++q) s += exp(f(q) - mx);
    return log(s) + mx;
  };
  for (int w = 1; w < N; ++w) {
    for (int i = tid; i + w < N; i += kT) {
      const int j = i + w;
      const double fold = red([&](int q) { return cr[i * N + i + q] + cl[(i + 1 + q) * N + j]; }, w);
      ir[i * N + j] = (double)th[i * N + j] + fold;
      il[i * N + j] = (double)th[j * N + i] + fold;
      cr[i * N + j] = red([&](int q) { return ir[i * N + i + 1 + q] + cr[(i + 1 + q) * N + j]; }, w);
      cl[i * N + j] = red([&](int q) { return cl[i * N + i + q] + il[(i + q) * N + j]; }, w);
    }
    __syncthreads();
  }
  for (int e = tid; e < num * N; e += kT) heads_all[(size_t)b * num * N + e] = -1;
  __syncthreads();
  if (tid != 0) return;
  // pick: first max of w (+ g) (spanning.py:287, numerics.py:162-168)
  int64_t pos = 0;
  auto choose = [&](auto f, int cnt) -> int {
    Pick p{ninfd(), -1};
    for (int q = 0; q < cnt; ++q) {
      const double v = f(q);
      if (kMax) {
        if (p.idx < 0 || v > p.best) p = Pick{v, q};
      } else {
        pick_add(p, v, g[pos + q], q);
      }
    }
    if (!kMax) pos += cnt;
    return p.idx < 0 ? 0 : p.idx;
  };
  double zroot = ninfd();
  if (single) {
    for (int c = 1; c <= n; ++c) zroot = fmax(zroot, (double)th[c] + cl[1 * N + c] + cr[c * N + n]);
  } else {
    zroot = cr[n];
  }
  const bool alive = zroot > ninfd();
  status[b] = alive ? SDB_ST_OK : SDB_ST_VACUOUS;
  extern __shared__ int estk[];  // walk stack [3][8 (n+2)] (dynamic), thread 0 only
  int* sk = estk;
  int* si = estk + 8 * (n + 2);
  int* sj = estk + 16 * (n + 2);
  if (alive) {
    for (int r = 0; r < num; ++r) {
      int32_t* heads = heads_all + ((size_t)b * num + r) * N;
      int top = 0;
      if (single) {
        const int c = 1 + choose([&](int q) { return (double)th[q + 1] + cl[1 * N + q + 1] + cr[(q + 1) * N + n]; }, n);
        heads[c] = 0;
        sk[top] = 1; si[top] = 1; sj[top++] = c;  // ("cl", 1, c)
        sk[top] = 0; si[top] = c; sj[top++] = n;  // ("cr", c, n)
      } else {
        sk[top] = 0; si[top] = 0; sj[top++] = n;
      }
      while (top > 0) {
        --top;
        const int kind = sk[top], i = si[top], j = sj[top];
        if (i == j) continue;
        if (kind == 0) {  // cr
          const int k = i + 1 + choose([&](int q) { return ir[i * N + i + 1 + q] + cr[(i + 1 + q) * N + j]; }, j - i);
          sk[top] = 2; si[top] = i; sj[top++] = k;
          sk[top] = 0; si[top] = k; sj[top++] = j;
        } else if (kind == 1) {  // cl
          const int k = i + choose([&](int q) { return cl[i * N + i + q] + il[(i + q) * N + j]; }, j - i);
          sk[top] = 1; si[top] = i; sj[top++] = k;
          sk[top] = 3; si[top] = k; sj[top++] = j;
        } else {
          if (kind == 2) heads[j] = i; else heads[i] = j;
          const int k = i + choose([&](int q) { return cr[i * N + i + q] + cl[(i + 1 + q) * N + j]; }, j - i);
          sk[top] = 0; si[top] = i; sj[top++] = k;
          sk[top] = 1; si[top] = k + 1; sj[top++] = j;
        }
      }
    }
  }
  used[b] = (int32_t)pos;
}

}  // namespace

// ------------------------------------------------------------------ C-ABI

extern "C" size_t sdb_chain_sample_workspace(int64_t B, int32_t n, int32_t m) {
  return (size_t)B * n * m * sizeof(double);
}
extern "C" int sdb_chain_sample(const float* init, const float* trans, int64_t B, int32_t n, int32_t m,
                                const double* noise, int64_t noise_per_instance, int32_t num, int32_t* tags,
                                int32_t* used, int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  if (B < 0 || n < 1 || m < 1 || num < 1) return SDB_ERR_ARG;
  if (m > 1024) return SDB_ERR_UNSUPPORTED;
  if (!init || (n > 1 && !trans) || !noise || !tags || !used || !status) return SDB_ERR_ARG;
  if (noise_per_instance < (int64_t)num * n * m) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!workspace || ws_bytes < sdb_chain_sample_workspace(B, n, m)) return SDB_ERR_WORKSPACE;
  const int thr = ((m + 31) / 32) * 32;
  chain_sample_kernel<<<(unsigned)B, thr, 0, (cudaStream_t)stream>>>(init, trans, n, m, noise, noise_per_instance, num,
                                                                     (double*)workspace, tags, used, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" size_t sdb_nw_sample_workspace(int64_t B, int32_t n, int32_t m) {
  return (size_t)B * (n + 1) * (m + 1) * sizeof(double);
}
extern "C" int sdb_nw_sample(const float* theta, int64_t B, int32_t n, int32_t m, const double* noise,
                             int64_t noise_per_instance, int32_t num, int8_t* path, int32_t* used, int32_t* status,
                             void* workspace, size_t ws_bytes, void* stream) {
  if (B < 0 || n < 0 || m < 0 || num < 1) return SDB_ERR_ARG;
  if (!theta || !noise || !path || !used || !status) return SDB_ERR_ARG;
  if (noise_per_instance < (int64_t)num * 3 * (n + m)) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!workspace || ws_bytes < sdb_nw_sample_workspace(B, n, m)) return SDB_ERR_WORKSPACE;
  nw_sample_kernel<<<(unsigned)B, kT, 0, (cudaStream_t)stream>>>(theta, n, m, noise, noise_per_instance, num,
                                                                (double*)workspace, path, used, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" size_t sdb_ctc_sample_workspace(int64_t B, int32_t T, int32_t V, int32_t L) {
  return (size_t)B * T * (2 * L + 1) * sizeof(double);
}
extern "C" int sdb_ctc_sample(const float* frame_potentials, const int32_t* targets, int64_t B, int32_t T, int32_t V,
                              int32_t L, const double* noise, int64_t noise_per_instance, int32_t num,
                              int32_t* states, int32_t* used, int32_t* status, void* workspace, size_t ws_bytes,
                              void* stream) {
  if (B < 0 || T < 1 || V < 2 || L < 0 || num < 1) return SDB_ERR_ARG;
  if (!frame_potentials || (L > 0 && !targets) || !noise || !states || !used || !status) return SDB_ERR_ARG;
  if (noise_per_instance < (int64_t)num * (2 + 3 * (int64_t)(T - 1))) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!workspace || ws_bytes < sdb_ctc_sample_workspace(B, T, V, L)) return SDB_ERR_WORKSPACE;
  ctc_sample_kernel<<<(unsigned)B, kT, 0, (cudaStream_t)stream>>>(frame_potentials, targets, T, V, L, noise,
                                                                 noise_per_instance, num, (double*)workspace, states,
                                                                 used, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" size_t sdb_tree_sample_workspace(int64_t B, int32_t n, int32_t m) {
  return (size_t)B * n * n * sizeof(double);
}
extern "C" int sdb_tree_sample(const float* span_potentials, int64_t B, int32_t n, int32_t m, const double* noise,
                               int64_t noise_per_instance, int32_t num, int32_t* labels, int32_t* used,
                               int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  if (B < 0 || n < 1 || m < 1 || num < 1) return SDB_ERR_ARG;
  if (n > 8192) return SDB_ERR_UNSUPPORTED;
  if (!span_potentials || !noise || !labels || !used || !status) return SDB_ERR_ARG;
  if (noise_per_instance < (int64_t)num * ((2 * n - 1) * (int64_t)m + (int64_t)n * n)) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!workspace || ws_bytes < sdb_tree_sample_workspace(B, n, m)) return SDB_ERR_WORKSPACE;
  const size_t stk = (size_t)4 * n * sizeof(int);
  if (sdb_set_smem((const void*)tree_sample_kernel, stk) != cudaSuccess) return SDB_ERR_CUDA;
  tree_sample_kernel<<<(unsigned)B, kT, stk, (cudaStream_t)stream>>>(span_potentials, n, m, noise, noise_per_instance,
                                                                  num, (double*)workspace, labels, used, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

extern "C" size_t sdb_eisner_decode_workspace(int64_t B, int32_t n) {
  return (size_t)B * 4 * (n + 1) * (n + 1) * sizeof(double);
}
extern "C" int sdb_eisner_decode(const float* adjacency, int64_t B, int32_t n, int32_t single_root,
                                 const double* noise, int64_t noise_per_instance, int32_t num, int32_t* heads,
                                 int32_t* used, int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  if (B < 0 || n < 1 || num < 1) return SDB_ERR_ARG;
  if (n > 2000) return SDB_ERR_UNSUPPORTED;
  if (!adjacency || !heads || !used || !status) return SDB_ERR_ARG;
  if (noise && noise_per_instance < (int64_t)num * (n + 4 * (int64_t)(n + 1) * (n + 1))) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!workspace || ws_bytes < sdb_eisner_decode_workspace(B, n)) return SDB_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t stk = (size_t)24 * (n + 2) * sizeof(int);
  if (sdb_set_smem(noise ? (const void*)eisner_decode_kernel<false> : (const void*)eisner_decode_kernel<true>, stk) !=
      cudaSuccess)
    return SDB_ERR_CUDA;
  if (noise)
    eisner_decode_kernel<false><<<(unsigned)B, kT, stk, s>>>(adjacency, n, single_root, noise, noise_per_instance, num,
                                                            (double*)workspace, heads, used, status);
  else
    eisner_decode_kernel<true><<<(unsigned)B, kT, stk, s>>>(adjacency, n, single_root, nullptr, 0, num,
                                                           (double*)workspace, heads, used, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

// ================================================================ Wilson
// spanning.py:531-558 (wilson_sample_arcs): loop-erased random walks toward
// the growing tree, one categorical pick per step over the dependent's
// incoming column (n+1 Gumbel draws per step).  Warp per instance; the walk
// state lives in the workspace so that a launch that runs out of stream
// (status 3) resumes where it stopped once the caller supplies the next
// chunk of the SAME Gumbel stream.
namespace {
struct WilsonState {
  int start, u, phase, pad;
  long long steps, used;
};

__global__ void wilson_kernel(int64_t B, const float* __restrict__ adj_all, int n, const double* __restrict__ noise_all,
                              int64_t cap, long long step_cap, WilsonState* __restrict__ st_all,
                              int32_t* __restrict__ parent_all, int8_t* __restrict__ in_tree_all,
                              int32_t* __restrict__ status) {
  const int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= B || status[b] != 3) return;  // 3 = walk in progress
  const int N = n + 1;
  const float* adj = adj_all + (size_t)b * N * N;
  const double* g = noise_all + (size_t)b * cap;
  WilsonState s = st_all[b];
  int32_t* parent = parent_all + (size_t)b * N;
  int8_t* in_tree = in_tree_all + (size_t)b * N;
  long long pos = 0;
  while (s.start <= n) {
    if (s.phase == 0) {
      if (in_tree[s.u]) {
        s.phase = 1;
        s.u = s.start;
        continue;
      }
      if (pos + N > cap) break;  // need the next chunk of the stream
      if (++s.steps > step_cap) {
        if (lane == 0) status[b] = 4;  // SamplerStepLimit
        s.steps = step_cap;
        break;
      }
      double best = ninfd();
      int arg = -1;
      for (int h = lane; h < N; h += 32) {
        const double w = (double)adj[(size_t)h * N + s.u];
        if (w > ninfd()) {
          const double v = w + g[pos + h];
          if (arg < 0 || v > best) {
            best = v;
            arg = h;
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, arg, o);
        if (oi >= 0 && (arg < 0 || ov > best || (ov == best && oi < arg))) {
          best = ov;
          arg = oi;
        }
      }
      pos += N;
      if (lane == 0) parent[s.u] = arg;
      __syncwarp();
      s.u = arg;
    } else {
      if (!in_tree[s.u]) {
        if (lane == 0) in_tree[s.u] = 1;
        __syncwarp();
        s.u = parent[s.u];
        continue;
      }
      ++s.start;
      s.u = s.start;
      s.phase = 0;
    }
  }
  s.used += pos;
  if (lane == 0) {
    st_all[b] = s;
    if (s.start > n) status[b] = SDB_ST_OK;
  }
}
}  // namespace

extern "C" size_t sdb_wilson_workspace(int64_t B, int32_t n) {
  return (size_t)B * (sizeof(WilsonState) + (size_t)(n + 1) * 5 + 16);
}

// One resumable pass of Wilson's algorithm.  On the first call (*status[b]
// != 3 on entry is taken as "start": status must be set to 3 by the caller
// together with a zeroed workspace, see sdb_wilson_begin).  noise [B, cap]
// holds the next cap draws of each instance's stream; used [B] (int64) returns
// how many were consumed in this pass; status: 0 done, 3 needs the next
// chunk, 4 step cap exceeded.  parent [B, n+1] is valid once status == 0.
extern "C" int sdb_wilson_step(const float* adjacency, int64_t B, int32_t n, const double* noise, int64_t cap,
                               int64_t step_cap, int32_t* parent, int64_t* used, int32_t* status, void* workspace,
                               size_t ws_bytes, void* stream) {
  if (B < 0 || n < 1 || cap < 0) return SDB_ERR_ARG;
  if (!adjacency || !noise || !parent || !used || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!workspace || ws_bytes < sdb_wilson_workspace(B, n)) return SDB_ERR_WORKSPACE;
  WilsonState* st = (WilsonState*)workspace;
  int8_t* in_tree = (int8_t*)(st + B);
  cudaStream_t s = (cudaStream_t)stream;
  wilson_kernel<<<(unsigned)((B + 3) / 4), 128, 0, s>>>(B, adjacency, n, noise, cap, (long long)step_cap, st, parent,
                                                        in_tree, status);
  SDB_CHECK_LAUNCH();
  // used[b] = cumulative draws consumed (the caller diffs successive values)
  if (cudaMemcpy2DAsync(used, sizeof(int64_t), (char*)st + offsetof(WilsonState, used), sizeof(WilsonState),
                        sizeof(int64_t), (size_t)B, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return SDB_ERR_CUDA;
  return SDB_OK;
}

// Initialise the walk state: root (and the optional pre-sampled root child)
// in the tree, status 3 for every instance.
namespace {
__global__ void wilson_begin_kernel(int n, int64_t B, const int32_t* __restrict__ child, WilsonState* st,
                                    int32_t* __restrict__ parent_all, int8_t* __restrict__ in_tree_all,
                                    int32_t* __restrict__ status) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int N = n + 1;
  for (int x = 0; x < N; ++x) {
    parent_all[(size_t)b * N + x] = -1;
    in_tree_all[(size_t)b * N + x] = (x == 0);
  }
  if (child) {
    const int c = child[b];
    parent_all[(size_t)b * N + c] = 0;
    in_tree_all[(size_t)b * N + c] = 1;
  }
  st[b] = WilsonState{1, 1, 0, 0, 0, 0};
  status[b] = 3;
}
}  // namespace

extern "C" int sdb_wilson_begin(int64_t B, int32_t n, const int32_t* root_child, int32_t* parent, int32_t* status,
                                void* workspace, size_t ws_bytes, void* stream) {
  if (B < 0 || n < 1 || !parent || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!workspace || ws_bytes < sdb_wilson_workspace(B, n)) return SDB_ERR_WORKSPACE;
  WilsonState* st = (WilsonState*)workspace;
  wilson_begin_kernel<<<(unsigned)((B + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      n, B, root_child, st, parent, (int8_t*)(st + B), status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

// =========================================================== semi-Markov
// chain.py:250-265 (alpha: lse over (width, prev) flattened width-major) and
// 330-344 (semi_markov_sample).  Thread per label for the chart; thread 0 walks.
namespace {
__global__ void __launch_bounds__(kT) semimarkov_sample_kernel(const float* __restrict__ th_all, int n, int s, int m,
                                                               const double* __restrict__ noise_all, int64_t cap,
                                                               int num, double* __restrict__ al_all,
                                                               int32_t* __restrict__ seg_all,
                                                               int32_t* __restrict__ nseg_all,
                                                               int32_t* __restrict__ used,
                                                               int32_t* __restrict__ status) {
  const int b = blockIdx.x, tid = threadIdx.x;
  const float* th = th_all + (size_t)b * n * s * m * m;  // [start][w-1][prev][label]
  double* al = al_all + (size_t)b * (n + 1) * m;
  const double* g = noise_all + (size_t)b * cap;
  int bad = 0;
  for (int e = tid; e < n * s * m * m; e += kT) bad |= bad_input(th[e]);
  const int anybad = __syncthreads_or(bad);
  if (anybad) {
    if (tid == 0) {
      status[b] = SDB_ST_INVALID;
      used[b] = 0;
    }
    return;
  }
  for (int l = tid; l < m; l += kT) al[l] = (l == 0) ? 0.0 : ninfd();
  __syncthreads();
  auto TH = [&](int st, int w, int p, int l) { return (double)th[(((size_t)st * s + w - 1) * m + p) * m + l]; };
  for (int t = 1; t <= n; ++t) {
    for (int l = tid; l < m; l += kT) {
      double mx = ninfd();
      const int W = min(s, t);
      for (int w = 1; w <= W; ++w)
        for (int p = 0; p < m; ++p) mx = fmax(mx, al[(size_t)(t - w) * m + p] + TH(t - w, w, p, l));
      double sm = 0.0;
      if (mx != ninfd())
        for (int w = 1; w <= W; ++w)
          for (int p = 0; p < m; ++p) sm += exp(al[(size_t)(t - w) * m + p] + TH(t - w, w, p, l) - mx);
      al[(size_t)t * m + l] = lse2(mx, sm);
    }
    __syncthreads();
  }
  if (tid != 0) return;
  bool alive = false;
  for (int l = 0; l < m; ++l) alive |= al[(size_t)n * m + l] > ninfd();
  status[b] = alive ? SDB_ST_OK : SDB_ST_VACUOUS;
  int64_t pos = 0;
  if (alive) {
    for (int r = 0; r < num; ++r) {
      int32_t* seg = seg_all + ((size_t)b * num + r) * n * 4;
      int cnt = 0;
      Pick p0{ninfd(), -1};
      for (int l = 0; l < m; ++l) pick_add(p0, al[(size_t)n * m + l], g[pos + l], l);
      pos += m;
      int t = n, l = p0.idx;
      while (t > 0) {
        const int W = min(s, t);
        Pick q{ninfd(), -1};
        for (int w = 1; w <= W; ++w)
          for (int p = 0; p < m; ++p) {
            const int f = (w - 1) * m + p;
            pick_add(q, al[(size_t)(t - w) * m + p] + TH(t - w, w, p, l), g[pos + f], f);
          }
        pos += (int64_t)W * m;
        const int w = 1 + q.idx / m, p = q.idx % m;
        seg[4 * cnt + 0] = t - w;
        seg[4 * cnt + 1] = w;
        seg[4 * cnt + 2] = p;
        seg[4 * cnt + 3] = l;
        ++cnt;
        t -= w;
        l = p;
      }
      nseg_all[(size_t)b * num + r] = cnt;
    }
  }
  used[b] = (int32_t)pos;
}
}  // namespace

extern "C" size_t sdb_semimarkov_sample_workspace(int64_t B, int32_t n, int32_t s, int32_t m) {
  return (size_t)B * (n + 1) * m * sizeof(double);
}

/* segments [B,num,n,4] (start, width, prev, label) in walk order (last
 * segment first), nseg [B,num]. */
extern "C" int sdb_semimarkov_sample(const float* segment_potentials, int64_t B, int32_t n, int32_t s, int32_t m,
                                     const double* noise, int64_t noise_per_instance, int32_t num, int32_t* segments,
                                     int32_t* nseg, int32_t* used, int32_t* status, void* workspace, size_t ws_bytes,
                                     void* stream) {
  if (B < 0 || n < 1 || s < 1 || m < 1 || num < 1) return SDB_ERR_ARG;
  if (!segment_potentials || !noise || !segments || !nseg || !used || !status) return SDB_ERR_ARG;
  if (noise_per_instance < (int64_t)num * ((int64_t)n * s * m + m)) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!workspace || ws_bytes < sdb_semimarkov_sample_workspace(B, n, s, m)) return SDB_ERR_WORKSPACE;
  semimarkov_sample_kernel<<<(unsigned)B, kT, 0, (cudaStream_t)stream>>>(segment_potentials, n, s, m, noise,
                                                                        noise_per_instance, num, (double*)workspace,
                                                                        segments, nseg, used, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
