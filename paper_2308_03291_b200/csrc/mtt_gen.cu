// Matrix-Tree theorem for n > 128 (the register-resident mtt.cu kernel's
// limit): same mathematics in fp64 with the Laplacian in the workspace
// (L2-resident), one 1024-thread CTA per instance.
//
// Reference: structdist spanning.py:90-175 and numerics.py:128-159 (see
// mtt.cu).  Gauss-Jordan in place with lazy pivot-row scaling: step k picks
// the pivot (multi-root: the diagonal -- column diagonal dominance,
// spanning.py:119; single root: partial pivoting, first maximum), stores the
// multipliers and the pivot row in shared memory, then every thread updates
// its share of the n x n matrix; three CTA barriers per step.  Feasibility
// (a spanning arborescence of finite weight exists) is checked structurally
// by breadth-first search, so an exactly singular Laplacian is -inf.
#include "common.cuh"

namespace {

constexpr int kGT = 1024;
constexpr int kGW = kGT / 32;
constexpr int kMaxGen = 2048;

template <typename TP>
__device__ bool reach_all(const TP* __restrict__ A, int n, int src, bool skip_root, uint8_t* seen, uint8_t* front,
                          int* flag) {
  const int N1 = n + 1;
  for (int v = threadIdx.x; v < N1; v += kGT) {
    seen[v] = (v == src);
    front[v] = (v == src);
  }
  __syncthreads();
  for (int it = 0; it < N1; ++it) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int d = threadIdx.x; d < N1; d += kGT) {
      if (seen[d] || d == 0) continue;
      for (int h = skip_root ? 1 : 0; h < N1; ++h) {
        if (front[h] && h != d && !((double)__ldg(A + (size_t)h * N1 + d) == ninfd())) {
          seen[d] = 2;  // reached this round
          *flag = 1;
          break;
        }
      }
    }
    __syncthreads();
    const int grew = *flag;
    for (int v = threadIdx.x; v < N1; v += kGT) {
      front[v] = (seen[v] == 2);
      if (seen[v] == 2) seen[v] = 1;
    }
    __syncthreads();
    if (!grew) break;
  }
  int miss = 0;
  for (int d = 1 + threadIdx.x; d < N1; d += kGT) miss |= !seen[d];
  return !__syncthreads_or(miss);
}

template <typename TP, typename M>  // adjacency / marginal types (float64 = exact mode)
__global__ void __launch_bounds__(kGT) mtt_gen_kernel(const TP* __restrict__ adj_all, int n, int single,
                                                      double* __restrict__ wsL, double* __restrict__ wsI,
                                                      double* __restrict__ logz, M* __restrict__ marg_all,
                                                      int32_t* __restrict__ status) {
  extern __shared__ __align__(16) double smd[];
  double* f = smd;               // [n] multipliers
  double* prow = f + n;          // [n] pivot row
  double* piv = prow + n;        // [n] pivots
  double* rowmag = piv + n;      // [n]
  double* shift = rowmag + n;             // [n] (column max, exact in either precision)
  int* perm = (int*)(shift + n);          // [n]
  int* qinv = perm + n;                   // [n]
  uint8_t* used = (uint8_t*)(qinv + n);   // [n]
  uint8_t* seen = used + n + 1;           // [n+1]
  uint8_t* front = seen + n + 1;          // [n+1]
  __shared__ double redv[kGW];
  __shared__ int redi[kGW];
  __shared__ int flag, bad_s, vac_s, pk_s;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N1 = n + 1;
  const TP* A = adj_all + (size_t)b * N1 * N1;
  double* L = wsL + (size_t)b * n * n;
  double* I = wsI + (size_t)b * n * n;
  if (tid == 0) { bad_s = 0; vac_s = 0; }
  __syncthreads();
  for (int e = tid; e < N1 * N1; e += kGT)
    if (bad_value(__ldg(A + e))) bad_s = 1;
  // column shifts (spanning.py:90-103)
  for (int d = tid; d < n; d += kGT) {
    double mx = ninfd();
    for (int h = 0; h <= n; ++h)
      if (h != d + 1) mx = fmax(mx, (double)__ldg(A + (size_t)h * N1 + d + 1));
    shift[d] = mx;
    if (mx == ninfd()) vac_s = 1;
  }
  __syncthreads();
  bool feasible = !bad_s && !vac_s;
  if (feasible) {
    if (!single) {
      feasible = reach_all(A, n, 0, false, seen, front, &flag);
    } else {
      feasible = false;
      for (int c = 1; c <= n && !feasible; ++c) {
        if ((double)__ldg(A + c) == ninfd()) continue;
        feasible = reach_all(A, n, c, true, seen, front, &flag);
      }
    }
  }
  if (!feasible) {
    if (tid == 0) {
      status[b] = bad_s ? SDB_ST_INVALID : SDB_ST_VACUOUS;
      logz[b] = ninfd();
    }
    if (marg_all)
      for (int e = tid; e < N1 * N1; e += kGT) marg_all[(size_t)b * N1 * N1 + e] = (M)0;
    return;
  }
  // Laplacian (spanning.py:106-120): column c = dependent c+1, row r = head r+1
  for (int e = tid; e < n * n; e += kGT) {
    const int r = e / n, c = e - r * n;
    double v;
    if (single && r == 0) {
      v = exp((double)__ldg(A + c + 1) - (double)shift[c]);
    } else if (r == c) {
      double s = 0.0;
      for (int h = single ? 1 : 0; h <= n; ++h)
        if (h != c + 1) s += exp((double)__ldg(A + (size_t)h * N1 + c + 1) - (double)shift[c]);
      v = s;
    } else {
      v = -exp((double)__ldg(A + (size_t)(r + 1) * N1 + c + 1) - (double)shift[c]);
    }
    L[e] = v;
  }
  __syncthreads();
  for (int r = warp; r < n; r += kGW) {  // original row magnitudes (numerics.py:143)
    double mx = 0.0;
    for (int c = lane; c < n; c += 32) mx = fmax(mx, fabs(L[(size_t)r * n + c]));
    mx = warp_maxd(mx);
    if (lane == 0) rowmag[r] = mx;
  }
  for (int r = tid; r < n; r += kGT) used[r] = 0;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    int p = k;
    if (single) {  // argmax |L[r][k]| over unused rows, first index on ties
      double bv = -1.0;
      int br = 0x7fffffff;
      for (int r = tid; r < n; r += kGT) {
        const double v = used[r] ? -1.0 : fabs(L[(size_t)r * n + k]);
        if (v > bv) { bv = v; br = r; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int orr = __shfl_xor_sync(0xffffffffu, br, o);
        if (ov > bv || (ov == bv && orr < br)) { bv = ov; br = orr; }
      }
      if (lane == 0) { redv[warp] = bv; redi[warp] = br; }
      __syncthreads();
      if (tid == 0) {
        double v = redv[0];
        int rr = redi[0];
        for (int w = 1; w < kGW; ++w)
          if (redv[w] > v || (redv[w] == v && redi[w] < rr)) { v = redv[w]; rr = redi[w]; }
        pk_s = rr;
      }
      __syncthreads();
      p = pk_s;
    }
    const double pv = L[(size_t)p * n + k];
    for (int c = tid; c < n; c += kGT) prow[c] = L[(size_t)p * n + c];
    for (int r = tid; r < n; r += kGT) f[r] = (r == p) ? 0.0 : L[(size_t)r * n + k] / pv;
    if (tid == 0) {
      piv[k] = pv;
      perm[k] = p;
      used[p] = 1;
    }
    __syncthreads();
    for (int e = tid; e < n * n; e += kGT) {
      const int r = e / n, c = e - r * n;
      const double v = L[e];
      L[e] = (c == k) ? ((r == p) ? 1.0 : -f[r]) : fma(-f[r], prow[c], v);
    }
    __syncthreads();
  }
  // log|det|, sign, singular pivots (numerics.py:140-159)
  double lg = 0.0;
  int neg = 0, sing = 0, inv = 0;
  for (int k = tid; k < n; k += kGT) {
    const double m = fabs(piv[k]);
    sing |= !(m > 1e-12 * fmax(rowmag[perm[k]], 1e-30));
    lg += log(m) + (double)shift[k];
    neg ^= piv[k] < 0.0;
    for (int j = k + 1; j < n; ++j) inv ^= (perm[j] < perm[k]);
  }
  for (int o = 16; o > 0; o >>= 1) lg += __shfl_xor_sync(0xffffffffu, lg, o);
  const int negs = __syncthreads_count(neg), invs = __syncthreads_count(inv), anys = __syncthreads_or(sing);
  if (lane == 0) redv[warp] = lg;
  __syncthreads();
  bool vac = false;
  {
    double t = 0.0;
    for (int w = 0; w < kGW; ++w) t += redv[w];
    vac = anys || ((negs + invs) & 1);
    if (tid == 0) {
      logz[b] = vac ? ninfd() : t;
      status[b] = vac ? SDB_ST_VACUOUS : SDB_ST_OK;
    }
  }
  if (!marg_all) return;
  // inverse: A^{-1}[q_i][perm_j] = M[i][j] / piv[q_i], stored transposed: I[perm_j][q_i]
  for (int k = tid; k < n; k += kGT) qinv[perm[k]] = k;
  __syncthreads();
  for (int e = tid; e < n * n; e += kGT) {
    const int i = e / n, j = e - i * n, qi = qinv[i];
    I[(size_t)perm[j] * n + qi] = L[e] / piv[qi];
  }
  __syncthreads();
  M* mg = marg_all + (size_t)b * N1 * N1;
  for (int e = tid; e < N1 * N1; e += kGT) {
    const int h = e / N1, dep = e - h * N1;
    double v = 0.0;
    if (!vac && dep >= 1 && h != dep) {
      const int d = dep - 1;
      const double w = exp((double)__ldg(A + e) - (double)shift[d]);
      const double idd = I[(size_t)d * n + d];
      if (single) {
        if (h == 0) v = w * I[d];  // I[0 * n + d]
        else v = w * ((d != 0 ? idd : 0.0) - ((h - 1) != 0 ? I[(size_t)(h - 1) * n + d] : 0.0));
      } else {
        v = (h == 0) ? w * idd : w * (idd - I[(size_t)(h - 1) * n + d]);
      }
      v = fmin(fmax(v, 0.0), 1.0);  // spanning.py:175
    }
    mg[e] = (M)v;
  }
}

}  // namespace

size_t mtt_gen_workspace(int64_t B, int n) { return (size_t)B * n * n * 8 * 2 + 256; }

template <typename TP, typename M>
int mtt_gen_launch_t(const TP* adjacency, int64_t B, int n, int single, double* logz, M* marg, int32_t* status,
                     void* workspace, size_t ws_bytes, cudaStream_t s) {
  if (n > kMaxGen) return SDB_ERR_UNSUPPORTED;
  if (!workspace || ws_bytes < mtt_gen_workspace(B, n)) return SDB_ERR_WORKSPACE;
  const size_t smem = (size_t)n * (5 * 8 + 4 + 4 + 1) + 2 * (size_t)(n + 1) + 64;
  if (sdb_set_smem((const void*)mtt_gen_kernel<TP, M>, smem) != cudaSuccess) return SDB_ERR_CUDA;
  double* L = (double*)workspace;
  double* I = L + (size_t)B * n * n;
  mtt_gen_kernel<TP, M><<<(unsigned)B, kGT, smem, s>>>(adjacency, n, single, L, I, logz, marg, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

int mtt_gen_launch(const float* adjacency, int64_t B, int n, int single, double* logz, float* marg, int32_t* status,
                   void* workspace, size_t ws_bytes, cudaStream_t s) {
  return mtt_gen_launch_t<float, float>(adjacency, B, n, single, logz, marg, status, workspace, ws_bytes, s);
}

// ---- exact mode (float64 adjacency and marginals, any n)
extern "C" size_t sdb_mtt_f64_workspace(int64_t B, int32_t n) { return (B < 0 || n < 1) ? 0 : mtt_gen_workspace(B, n); }
extern "C" int sdb_mtt_f64(const double* adjacency, int64_t B, int32_t n, int32_t single_root, double* logz,
                           double* marg, int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  if (B < 0 || n < 1 || !adjacency || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  return mtt_gen_launch_t<double, double>(adjacency, B, n, single_root ? 1 : 0, logz, marg, status, workspace,
                                          ws_bytes, (cudaStream_t)stream);
}
