// Monotone alignment for shapes beyond the strip kernels' limit (m > 351):
// the reference recurrences (structdist alignment.py:62-167) on anti-diagonals,
// fp64, one CTA per instance.
//
// Diagonal d holds the cells (i, d - i), i in [max(0, d - m), min(n, d)]; its
// values depend only on diagonals d-1 and d-2, which live in shared memory
// (3 rotating buffers of min(n, m) + 1 doubles).  The forward pass keeps the
// full alpha grid in the workspace when a later pass needs it (marginals read
// alpha(src) while the backward pass walks the diagonals in reverse and emits
// exp(alpha(src) + theta + beta - log Z) cell by cell; the argmax walk reads
// the max-plus alpha).  One __syncthreads per diagonal.
#include "common.cuh"

namespace {

constexpr int kT = 512;

__device__ __forceinline__ double lse3d(double a, double b, double c) {
  const double M = fmax(a, fmax(b, c));
  if (M == ninfd()) return ninfd();
  return M + log(exp(a - M) + exp(b - M) + exp(c - M));
}

struct Diag {
  int n, m;
  __device__ int lo(int d) const { return d > m ? d - m : 0; }
  __device__ int hi(int d) const { return d < n ? d : n; }
};

// kMode 0: log Z; 1: log Z + marginals; 2: max-plus score + argmax path.
// T / M: potential and marginal types (float: the batched fp32 contract;
// double: the exact mode, float64 in and out like the reference)
template <int kMode, typename T, typename M>
__global__ void __launch_bounds__(kT) nw_gen_kernel(const T* __restrict__ theta, int n, int m,
                                                    double* __restrict__ ws_all, double* __restrict__ out,
                                                    M* __restrict__ marg_all, int8_t* __restrict__ path_all,
                                                    int32_t* __restrict__ status) {
  extern __shared__ __align__(16) double dbuf[];
  __shared__ int bad_s;
  __shared__ double z_s;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int n1 = n + 1, m1 = m + 1, L = min(n, m) + 1;
  const T* th = theta + (size_t)b * n1 * m1 * 3;
  double* A = kMode ? ws_all + (size_t)b * n1 * m1 : nullptr;
  double* dv[3] = {dbuf, dbuf + L, dbuf + 2 * L};
  const Diag D{n, m};
  auto Th = [&](int i, int j, int k) { return (double)__ldg(th + ((size_t)i * m1 + j) * 3 + k); };
  if (tid == 0) bad_s = 0;
  __syncthreads();
  {
    int bad = 0;
    for (size_t e = tid; e < (size_t)n1 * m1 * 3; e += kT) bad |= bad_value(__ldg(th + e));
    if (bad) bad_s = 1;
  }
  // forward (alignment.py:62-76; max-plus for the argmax, alignment.py:155-167)
  for (int d = 0; d <= n + m; ++d) {
    double* cur = dv[d % 3];
    const double* p1 = dv[(d + 2) % 3];  // d - 1
    const double* p2 = dv[(d + 1) % 3];  // d - 2
    const int lo = D.lo(d), hi = D.hi(d), lo1 = D.lo(d - 1), lo2 = D.lo(d - 2);
    for (int i = lo + tid; i <= hi; i += kT) {
      const int j = d - i;
      double a;
      if (d == 0) {
        a = 0.0;
      } else {
        const double c0 = (i > 0 && j > 0) ? p2[i - 1 - lo2] + Th(i, j, 0) : ninfd();
        const double c1 = (i > 0) ? p1[i - 1 - lo1] + Th(i, j, 1) : ninfd();
        const double c2 = (j > 0) ? p1[i - lo1] + Th(i, j, 2) : ninfd();
        a = kMode == 2 ? fmax(c0, fmax(c1, c2)) : lse3d(c0, c1, c2);
      }
      cur[i - lo] = a;
      if (kMode) A[(size_t)i * m1 + j] = a;
    }
    __syncthreads();
  }
  if (tid == 0) z_s = dv[(n + m) % 3][n - D.lo(n + m)];
  __syncthreads();
  const double z = z_s;
  const bool bad = bad_s != 0;
  if (tid == 0) {
    out[b] = z;
    status[b] = bad ? SDB_ST_INVALID : (z == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
  }
  if (kMode == 1) {
    M* mg = marg_all + (size_t)b * n1 * m1 * 3;
    const bool zok = !bad && z != ninfd();
    // backward (alignment.py:79-99) with the marginals of each finished cell
    for (int d = n + m; d >= 0; --d) {
      double* cur = dv[d % 3];
      const double* q1 = dv[(d + 1) % 3];  // d + 1
      const double* q2 = dv[(d + 2) % 3];  // d + 2
      const int lo = D.lo(d), hi = D.hi(d), lq1 = D.lo(d + 1), lq2 = D.lo(d + 2);
      for (int i = lo + tid; i <= hi; i += kT) {
        const int j = d - i;
        double bt;
        if (d == n + m) {
          bt = 0.0;
        } else {
          const double c0 = (i < n && j < m) ? Th(i + 1, j + 1, 0) + q2[i + 1 - lq2] : ninfd();
          const double c1 = (i < n) ? Th(i + 1, j, 1) + q1[i + 1 - lq1] : ninfd();
          const double c2 = (j < m) ? Th(i, j + 1, 2) + q1[i - lq1] : ninfd();
          bt = lse3d(c0, c1, c2);
        }
        cur[i - lo] = bt;
        M* o = mg + ((size_t)i * m1 + j) * 3;
        const double base = bt - z;
        o[0] = (M)((zok && i > 0 && j > 0) ? exp(A[(size_t)(i - 1) * m1 + j - 1] + Th(i, j, 0) + base) : 0.0);
        o[1] = (M)((zok && i > 0) ? exp(A[(size_t)(i - 1) * m1 + j] + Th(i, j, 1) + base) : 0.0);
        o[2] = (M)((zok && j > 0) ? exp(A[(size_t)i * m1 + j - 1] + Th(i, j, 2) + base) : 0.0);
      }
      __syncthreads();
    }
  }
  if (kMode == 2 && tid == 0 && !bad && z != ninfd()) {
    // walk back from (n, m), first maximum among DIAG, DOWN, RIGHT (alignment.py:121-140)
    int8_t* pb = path_all + (size_t)b * n1 * m1;
    int i = n, j = m;
    while (i != 0 || j != 0) {
      int k = -1;
      double best = 0.0;
      if (i > 0 && j > 0) { best = A[(size_t)(i - 1) * m1 + j - 1] + Th(i, j, 0); k = 0; }
      if (i > 0) {
        const double c = A[(size_t)(i - 1) * m1 + j] + Th(i, j, 1);
        if (k < 0 || c > best) { best = c; k = 1; }
      }
      if (j > 0) {
        const double c = A[(size_t)i * m1 + j - 1] + Th(i, j, 2);
        if (k < 0 || c > best) { best = c; k = 2; }
      }
      pb[(size_t)i * m1 + j] = (int8_t)k;
      if (k == 0) { --i; --j; } else if (k == 1) { --i; } else { --j; }
    }
  }
}

}  // namespace

constexpr int kNwGenMaxDiag = 8192;

bool nw_gen_ok(int n, int m) { return min(n, m) + 1 <= kNwGenMaxDiag; }

size_t nw_gen_workspace(int64_t B, int n, int m, int mode) {
  return mode ? (size_t)B * (n + 1) * (m + 1) * sizeof(double) + 256 : 0;
}

template <typename T, typename M>
int nw_gen_launch_t(int mode, const T* theta, int64_t B, int n, int m, void* ws, size_t ws_bytes, double* out, M* marg,
                    int8_t* path, int32_t* status, cudaStream_t s) {
  if (!nw_gen_ok(n, m)) return SDB_ERR_UNSUPPORTED;
  if (ws_bytes < nw_gen_workspace(B, n, m, mode) || (mode && !ws)) return SDB_ERR_WORKSPACE;
  const size_t smem = (size_t)3 * (min(n, m) + 1) * sizeof(double);
  const void* k = mode == 0 ? (const void*)nw_gen_kernel<0, T, M> : mode == 1 ? (const void*)nw_gen_kernel<1, T, M>
                                                                               : (const void*)nw_gen_kernel<2, T, M>;
  if (sdb_set_smem(k, smem) != cudaSuccess) return SDB_ERR_CUDA;
  double* w = (double*)ws;
  if (mode == 0) nw_gen_kernel<0, T, M><<<(unsigned)B, kT, smem, s>>>(theta, n, m, w, out, marg, path, status);
  if (mode == 1) nw_gen_kernel<1, T, M><<<(unsigned)B, kT, smem, s>>>(theta, n, m, w, out, marg, path, status);
  if (mode == 2) nw_gen_kernel<2, T, M><<<(unsigned)B, kT, smem, s>>>(theta, n, m, w, out, marg, path, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

int nw_gen_launch(int mode, const float* theta, int64_t B, int n, int m, void* ws, size_t ws_bytes, double* out,
                  float* marg, int8_t* path, int32_t* status, cudaStream_t s) {
  return nw_gen_launch_t<float, float>(mode, theta, B, n, m, ws, ws_bytes, out, marg, path, status, s);
}

// ---- exact mode (float64 potentials and marginals, any shape)
extern "C" size_t sdb_nw_fb_f64_workspace(int64_t B, int32_t n, int32_t m) {
  return (B < 0 || n < 1 || m < 1) ? 0 : nw_gen_workspace(B, n, m, 1);
}
extern "C" int sdb_nw_fb_f64(const double* theta, int64_t B, int32_t n, int32_t m, double* logz, double* marg,
                             int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  if (B < 0 || n < 1 || m < 1 || !theta || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  return nw_gen_launch_t<double, double>(marg ? 1 : 0, theta, B, n, m, workspace, ws_bytes, logz, marg, nullptr,
                                         status, (cudaStream_t)stream);
}
