// Tree-CRF CKY for sentences beyond the shared-memory chart kernels
// (n > 128): the reference's inside / outside / walk (structdist
// constituency.py:52-133) in fp64 with the charts in global memory, one CTA
// (32 warps) per instance, one warp per span of the current width, one
// __syncthreads per width.
#include "common.cuh"

namespace {

constexpr int kT = 1024;
constexpr int kW = kT / 32;

struct WLse {  // per-lane online log-sum-exp (or max), then a warp reduction
  double mx = ninfd(), s = 0.0;
  __device__ void add(double x, bool maxplus) {
    if (maxplus) { mx = fmax(mx, x); return; }
    if (x == ninfd()) return;
    if (x > mx) { s = s * exp(mx - x) + 1.0; mx = x; } else { s += exp(x - mx); }
  }
  __device__ double reduce(bool maxplus) {
    double M = mx;
    for (int o = 16; o > 0; o >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
    if (maxplus || M == ninfd()) return M;
    double t = (mx == ninfd()) ? 0.0 : s * exp(mx - M);
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    return M + log(t);
  }
};

// kMode 0: log Z; 1: log Z + marginals; 2: max-plus score + best tree labels
template <int kMode, typename TP, typename M>  // TP / M: potential / marginal types (float64 = exact mode)
__global__ void __launch_bounds__(kT) tree_gen_kernel(const TP* __restrict__ sp_all, int n, int m,
                                                      double* __restrict__ ws_all, double* __restrict__ out,
                                                      M* __restrict__ marg_all, int32_t* __restrict__ lab_all,
                                                      int32_t* __restrict__ status) {
  __shared__ int bad_s;
  constexpr bool kMax = kMode == 2;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t nn = (size_t)n * n;
  const TP* sp = sp_all + (size_t)b * nn * m;
  double* S = ws_all + (size_t)b * 3 * nn;  // label fold
  double* I = S + nn;                       // inside
  double* O = I + nn;                       // outside (marginals) / walk stack (argmax)
  if (tid == 0) bad_s = 0;
  __syncthreads();
  {
    int bad = 0;
    for (size_t e = tid; e < nn * m; e += kT) bad |= bad_value(__ldg(sp + e));
    if (bad) bad_s = 1;
  }
  // label fold (constituency.py:55), one warp per span
  for (size_t e = warp; e < nn; e += kW) {
    const int i = (int)(e / n), j = (int)(e % n);
    if (i > j) continue;
    WLse r;
    for (int l = lane; l < m; l += 32) r.add((double)__ldg(sp + e * m + l), kMax);
    const double v = r.reduce(kMax);
    if (lane == 0) {
      S[e] = v;
      if (i == j) I[e] = v;
    }
  }
  __syncthreads();
  // inside by width (constituency.py:56-63)
  for (int w = 2; w <= n; ++w) {
    for (int i = warp; i + w - 1 < n; i += kW) {
      const int j = i + w - 1;
      WLse r;
      for (int k = i + lane; k < j; k += 32) r.add(I[(size_t)i * n + k] + I[(size_t)(k + 1) * n + j], kMax);
      const double v = r.reduce(kMax);
      if (lane == 0) I[(size_t)i * n + j] = S[(size_t)i * n + j] + v;
    }
    __syncthreads();
  }
  const double z = I[n - 1];
  const bool bad = bad_s != 0;
  if (tid == 0) {
    out[b] = z;
    status[b] = bad ? SDB_ST_INVALID : (z == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
  }
  if (kMode == 1) {
    M* mg = marg_all + (size_t)b * nn * m;
    const bool zok = !bad && z != ninfd();
    for (size_t e = tid; e < nn; e += kT) O[e] = ninfd();
    __syncthreads();
    if (tid == 0) O[n - 1] = 0.0;
    __syncthreads();
    // outside by width, widest first (constituency.py:83-97)
    for (int w = n - 1; w >= 1; --w) {
      for (int i = warp; i + w - 1 < n; i += kW) {
        const int j = i + w - 1;
        WLse r;
        for (int pj = j + 1 + lane; pj < n; pj += 32)
          r.add(O[(size_t)i * n + pj] + S[(size_t)i * n + pj] + I[(size_t)(j + 1) * n + pj], false);
        for (int pi = lane; pi < i; pi += 32)
          r.add(O[(size_t)pi * n + j] + S[(size_t)pi * n + j] + I[(size_t)pi * n + i - 1], false);
        const double v = r.reduce(false);
        if (lane == 0) O[(size_t)i * n + j] = v;
      }
      __syncthreads();
    }
    // labeled-span marginals (constituency.py:98-110)
    for (size_t e = tid; e < nn * m; e += kT) {
      const size_t c = e / m;
      const int i = (int)(c / n), j = (int)(c % n);
      double v = 0.0;
      if (zok && i <= j && I[c] != ninfd() && O[c] != ninfd())
        v = exp(O[c] + (I[c] - S[c]) + (double)__ldg(sp + e) - z);
      mg[e] = (M)v;
    }
  }
  if (kMode == 2 && tid == 0 && !bad && z != ninfd()) {
    // walk (constituency.py:113-133): first argmax label, first argmax split
    int32_t* lab = lab_all + (size_t)b * nn;
    int* stack = (int*)O;
    int top = 0;
    stack[top++] = n - 1;  // (0, n-1) encoded as i * n + j
    while (top > 0) {
      const int c = stack[--top], i = c / n, j = c % n;
      const TP* th = sp + (size_t)c * m;
      int bl = 0;
      for (int l = 1; l < m; ++l)
        if (th[l] > th[bl]) bl = l;
      lab[c] = bl;
      if (i == j) continue;
      int bk = i;
      double bv = I[(size_t)i * n + i] + I[(size_t)(i + 1) * n + j];
      for (int k = i + 1; k < j; ++k) {
        const double v = I[(size_t)i * n + k] + I[(size_t)(k + 1) * n + j];
        if (v > bv) { bv = v; bk = k; }
      }
      stack[top++] = i * n + bk;
      stack[top++] = (bk + 1) * n + j;
    }
  }
}

}  // namespace

bool tree_gen_ok(int n) { return n <= 8192; }

size_t tree_gen_workspace(int64_t B, int n) { return (size_t)B * 3 * n * n * sizeof(double) + 256; }

template <typename TP, typename M>
int tree_gen_launch_t(int mode, const TP* sp, int64_t B, int n, int m, void* ws, size_t ws_bytes, double* out,
                      M* marg, int32_t* labels, int32_t* status, cudaStream_t s) {
  if (!tree_gen_ok(n)) return SDB_ERR_UNSUPPORTED;
  const size_t need = tree_gen_workspace(B, n);
  bool own = false;
  if (!ws) {  // sdb_tree_viterbi has no workspace argument: stream-ordered scratch
    if (sdb_note(cudaMallocAsync(&ws, need, s)) != cudaSuccess) return SDB_ERR_CUDA;
    own = true;
  } else if (ws_bytes < need) {
    return SDB_ERR_WORKSPACE;
  }
  double* w = (double*)ws;
  if (mode == 2 && sdb_note(cudaMemsetAsync(labels, 0xff, (size_t)B * n * n * sizeof(int32_t), s)) != cudaSuccess)
    return SDB_ERR_CUDA;
  if (mode == 0) tree_gen_kernel<0, TP, M><<<(unsigned)B, kT, 0, s>>>(sp, n, m, w, out, marg, labels, status);
  if (mode == 1) tree_gen_kernel<1, TP, M><<<(unsigned)B, kT, 0, s>>>(sp, n, m, w, out, marg, labels, status);
  if (mode == 2) tree_gen_kernel<2, TP, M><<<(unsigned)B, kT, 0, s>>>(sp, n, m, w, out, marg, labels, status);
  SDB_CHECK_LAUNCH();
  if (own && sdb_note(cudaFreeAsync(ws, s)) != cudaSuccess) return SDB_ERR_CUDA;
  return SDB_OK;
}

int tree_gen_launch(int mode, const float* sp, int64_t B, int n, int m, void* ws, size_t ws_bytes, double* out,
                    float* marg, int32_t* labels, int32_t* status, cudaStream_t s) {
  return tree_gen_launch_t<float, float>(mode, sp, B, n, m, ws, ws_bytes, out, marg, labels, status, s);
}

// ---- exact mode (float64 span potentials and marginals)
extern "C" size_t sdb_tree_fb_f64_workspace(int64_t B, int32_t n, int32_t m) {
  (void)m;
  return (B < 0 || n < 1) ? 0 : tree_gen_workspace(B, n);
}
extern "C" int sdb_tree_fb_f64(const double* span_potentials, int64_t B, int32_t n, int32_t m, double* logz,
                               double* marg, int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  if (B < 0 || n < 1 || m < 1 || !span_potentials || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  if (!workspace) return SDB_ERR_WORKSPACE;
  return tree_gen_launch_t<double, double>(marg ? 1 : 0, span_potentials, B, n, m, workspace, ws_bytes, logz, marg,
                                           nullptr, status, (cudaStream_t)stream);
}
