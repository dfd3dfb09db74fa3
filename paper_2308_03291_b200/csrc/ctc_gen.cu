// CTC for lattices beyond the state-per-thread kernels (2L+1 > 1024 states or
// a vocabulary too large for the staged frame rows): the reference recurrences
// (structdist alignment.py:231-336) in fp64, one CTA per instance, states
// strided over the threads.
//
// The current and previous lattice rows live in shared memory; alpha is kept
// for every frame in the workspace when a later pass needs it (marginals:
// the backward pass emits exp(alpha + beta - log Z) per (frame, state) and
// scatter-adds it into the state's label with float atomics, as
// ctc_marginals does with its loop over labels; argmax: the walk re-reads the
// max-plus lattice with the reference's first-maximum ties).
#include "common.cuh"

namespace {

constexpr int kT = 1024;

__device__ __forceinline__ double lse3d(double a, double b, double c) {
  const double M = fmax(a, fmax(b, c));
  if (M == ninfd()) return ninfd();
  return M + log(exp(a - M) + exp(b - M) + exp(c - M));
}

struct Lab {
  const int32_t* tg;
  int S;
  __device__ int operator()(int s) const { return (s & 1) ? tg[s >> 1] : 0; }
  // s-2 -> s allowed (alignment.py:239-245)
  __device__ bool skip(int s) const {
    if (s < 2 || !(s & 1)) return false;
    return tg[s >> 1] != tg[(s >> 1) - 1];
  }
};

// kMode 0: log Z; 1: log Z + marginals [T][V]; 2: max-plus score + labels per frame
template <int kMode, typename TP, typename M>  // TP / M: potential / marginal types (float64 = exact mode)
__global__ void __launch_bounds__(kT) ctc_gen_kernel(const TP* __restrict__ fp_all, const int32_t* __restrict__ tg_all,
                                                     int T, int V, int L, double* __restrict__ ws_all,
                                                     double* __restrict__ out, M* __restrict__ marg_all,
                                                     int32_t* __restrict__ path_all, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) double rows[];  // [2][S]
  __shared__ int bad_s;
  __shared__ double z_s;
  __shared__ int fin_s;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int S = 2 * L + 1;
  const TP* fp = fp_all + (size_t)b * T * V;
  const Lab lab{tg_all + (size_t)b * L, S};
  double* A = kMode ? ws_all + (size_t)b * T * S : nullptr;
  auto E = [&](int t, int s) { return (double)__ldg(fp + (size_t)t * V + lab(s)); };
  if (tid == 0) bad_s = 0;
  __syncthreads();
  {
    int bad = 0;
    for (size_t e = tid; e < (size_t)T * V; e += kT) bad |= bad_value(__ldg(fp + e));
    for (int x = tid; x < L; x += kT) bad |= (lab.tg[x] < 1) | (lab.tg[x] >= V);
    if (bad) bad_s = 1;
  }
  __syncthreads();
  const bool bad = bad_s != 0;
  if (bad) {
    if (tid == 0) {
      out[b] = ninfd();
      status[b] = SDB_ST_INVALID;
    }
    return;  // labels may be out of range: do not index with them
  }
  // forward (alignment.py:248-260; max-plus 321-333)
  double* prv = rows;
  double* cur = rows + S;
  for (int s = tid; s < S; s += kT) {
    const double a = s <= 1 ? E(0, s) : ninfd();
    prv[s] = a;
    if (kMode) A[s] = a;
  }
  __syncthreads();
  for (int t = 1; t < T; ++t) {
    for (int s = tid; s < S; s += kT) {
      const double x0 = prv[s], x1 = s >= 1 ? prv[s - 1] : ninfd(), x2 = lab.skip(s) ? prv[s - 2] : ninfd();
      const double acc = kMode == 2 ? fmax(x0, fmax(x1, x2)) : lse3d(x0, x1, x2);
      const double a = acc + E(t, s);
      cur[s] = a;
      if (kMode) A[(size_t)t * S + s] = a;
    }
    __syncthreads();
    double* x = prv;
    prv = cur;
    cur = x;
  }
  if (tid == 0) {
    const double f1 = prv[S - 1], f2 = S > 1 ? prv[S - 2] : ninfd();
    double z;
    int fin = S - 1;
    if (kMode == 2) {
      z = f1;  // first maximum over the finals [S-1, S-2]
      if (S > 1 && f2 > f1) { z = f2; fin = S - 2; }
    } else {
      z = lse3d(f1, f2, ninfd());
    }
    z_s = z;
    fin_s = fin;
    out[b] = z;
    status[b] = z == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK;
  }
  __syncthreads();
  const double z = z_s;
  if (z == ninfd()) return;  // marginals were zeroed by the launcher; labels stay 0
  if (kMode == 1) {
    // backward (alignment.py:272-290) + posteriors scattered by label (291-301)
    M* mg = marg_all + (size_t)b * T * V;
    double* nxt = prv;  // beta[t+1]
    double* now = cur;
    // blank states (even s) share label 0: reduced per warp before the atomic
    auto emit = [&](int t, int s, double p, double& pb) {
      if (s & 1) {
        if (p > 0.0) atomicAdd(mg + (size_t)t * V + lab(s), (M)p);
      } else {
        pb += p;
      }
    };
    auto flush_blank = [&](int t, double pb) {
      for (int o = 16; o > 0; o >>= 1) pb += __shfl_xor_sync(0xffffffffu, pb, o);
      if ((tid & 31) == 0 && pb > 0.0) atomicAdd(mg + (size_t)t * V, (M)pb);
    };
    {
      double pb = 0.0;
      for (int s = tid; s < S; s += kT) {
        const double bt = (s == S - 1 || s == S - 2) ? 0.0 : ninfd();
        nxt[s] = bt;
        emit(T - 1, s, exp(A[(size_t)(T - 1) * S + s] + bt - z), pb);
      }
      flush_blank(T - 1, pb);
    }
    __syncthreads();
    for (int t = T - 2; t >= 0; --t) {
      double pb = 0.0;
      for (int s = tid; s < S; s += kT) {
        const double y0 = E(t + 1, s) + nxt[s];
        const double y1 = s + 1 < S ? E(t + 1, s + 1) + nxt[s + 1] : ninfd();
        const double y2 = (s + 2 < S && lab.skip(s + 2)) ? E(t + 1, s + 2) + nxt[s + 2] : ninfd();
        const double bt = lse3d(y0, y1, y2);
        now[s] = bt;
        emit(t, s, exp(A[(size_t)t * S + s] + bt - z), pb);
      }
      flush_blank(t, pb);
      __syncthreads();
      double* x = nxt;
      nxt = now;
      now = x;
    }
  }
  if (kMode == 2 && tid == 0) {
    // walk (alignment.py:304-318): predecessors [s, s-1, s-2], first maximum
    int32_t* path = path_all + (size_t)b * T;
    int s = fin_s;
    for (int t = T - 1; t >= 0; --t) {
      path[t] = lab(s);
      if (t == 0) break;
      const double* a = A + (size_t)(t - 1) * S;
      int best = s;
      double bv = a[s];
      if (s >= 1 && a[s - 1] > bv) { bv = a[s - 1]; best = s - 1; }
      if (lab.skip(s) && a[s - 2] > bv) { bv = a[s - 2]; best = s - 2; }
      s = best;
    }
  }
}

}  // namespace

constexpr int kCtcGenMaxS = 12 * 1024;

bool ctc_gen_ok(int L) { return 2 * L + 1 <= kCtcGenMaxS; }

size_t ctc_gen_workspace(int64_t B, int T, int L, int mode) {
  return mode ? (size_t)B * T * (2 * L + 1) * sizeof(double) + 256 : 0;
}

template <typename TP, typename M>
int ctc_gen_launch_t(int mode, const TP* fp, const int32_t* tg, int64_t B, int T, int V, int L, void* ws,
                     size_t ws_bytes, double* out, M* marg, int32_t* path, int32_t* status, cudaStream_t s) {
  if (!ctc_gen_ok(L)) return SDB_ERR_UNSUPPORTED;
  if (ws_bytes < ctc_gen_workspace(B, T, L, mode) || (mode && !ws)) return SDB_ERR_WORKSPACE;
  const size_t smem = (size_t)2 * (2 * L + 1) * sizeof(double);
  const void* k = mode == 0 ? (const void*)ctc_gen_kernel<0, TP, M>
                            : mode == 1 ? (const void*)ctc_gen_kernel<1, TP, M> : (const void*)ctc_gen_kernel<2, TP, M>;
  if (sdb_set_smem(k, smem) != cudaSuccess) return SDB_ERR_CUDA;
  double* w = (double*)ws;
  if (mode == 1 && sdb_note(cudaMemsetAsync(marg, 0, (size_t)B * T * V * sizeof(M), s)) != cudaSuccess)
    return SDB_ERR_CUDA;
  if (mode == 2 && sdb_note(cudaMemsetAsync(path, 0, (size_t)B * T * sizeof(int32_t), s)) != cudaSuccess)
    return SDB_ERR_CUDA;
  if (mode == 0) ctc_gen_kernel<0, TP, M><<<(unsigned)B, kT, smem, s>>>(fp, tg, T, V, L, w, out, marg, path, status);
  if (mode == 1) ctc_gen_kernel<1, TP, M><<<(unsigned)B, kT, smem, s>>>(fp, tg, T, V, L, w, out, marg, path, status);
  if (mode == 2) ctc_gen_kernel<2, TP, M><<<(unsigned)B, kT, smem, s>>>(fp, tg, T, V, L, w, out, marg, path, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

int ctc_gen_launch(int mode, const float* fp, const int32_t* tg, int64_t B, int T, int V, int L, void* ws,
                   size_t ws_bytes, double* out, float* marg, int32_t* path, int32_t* status, cudaStream_t s) {
  return ctc_gen_launch_t<float, float>(mode, fp, tg, B, T, V, L, ws, ws_bytes, out, marg, path, status, s);
}

// ---- exact mode (float64 frame potentials and marginals)
extern "C" size_t sdb_ctc_fb_f64_workspace(int64_t B, int32_t T, int32_t V, int32_t L) {
  (void)V;
  return (B < 0 || T < 1 || L < 0) ? 0 : ctc_gen_workspace(B, T, L, 1);
}
extern "C" int sdb_ctc_fb_f64(const double* frame_potentials, const int32_t* targets, int64_t B, int32_t T, int32_t V,
                              int32_t L, double* logz, double* marg, int32_t* status, void* workspace,
                              size_t ws_bytes, void* stream) {
  if (B < 0 || T < 1 || V < 1 || L < 0 || !frame_potentials || (L > 0 && !targets) || !logz || !status)
    return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  return ctc_gen_launch_t<double, double>(marg ? 1 : 0, frame_potentials, targets, B, T, V, L, workspace, ws_bytes,
                                          logz, marg, nullptr, status, (cudaStream_t)stream);
}
