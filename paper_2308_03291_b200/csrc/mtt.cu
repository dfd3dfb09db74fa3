// Non-projective spanning trees via the Matrix-Tree theorem: log-partition
// (log|det| of the root-augmented Laplacian) and edge marginals (inverse
// Laplacian).
//
// Reference: structdist spanning.py:90-175 (_shifted_exp_weights,
// _build_laplacian, mtt_log_partition, mtt_marginals) and numerics.py:128-159
// (signed_log_det: partial pivoting, singular when |pivot| <= 1e-12 * the
// pivot row's original max-abs; -inf when sign <= 0).
// Layout per instance: adjacency [n+1][n+1] fp32 (head, dependent).
//
// One CTA (512 threads) per instance, n <= 128 (padded to 128 with an
// identity block).  The 128x128 Laplacian lives in REGISTERS: warp w owns
// columns [8w, 8w+8), lane l owns rows [4l, 4l+4) -> 32 fp32 per thread.
// In-place Gauss-Jordan with implicit partial pivoting: step k picks the
// unused row p with max |a[p][k]| (a warp argmax inside the column's warp),
// broadcasts row p and column k through shared memory, and every thread does
// a register-blocked rank-1 update (32 FFMA per 12 shared loads).  Pivots
// equal the reference's LU pivots, so log|det| = sum log|pivot| (fp64) and the
// sign comes from the pivot signs and the permutation parity.  The result is
// the row/column-permuted inverse, scattered to shared memory as A^{-1}, from
// which the edge marginals are formed (spanning.py:152-175) and clipped.
#include "common.cuh"

namespace {

constexpr int kN = 128;
constexpr int kThreads = 512;

struct MttSmem {
  float* adj;     // [(n+1)*(n+1)]
  float* inv;     // [kN*kN] A^{-1}
  float* shift;   // [kN] column max s_d
  float* diag;    // [kN]
  float* rowmag;  // [kN]
  float* rowbuf;  // [2][kN]
  float* colbuf;  // [2][kN]
  int* perm;      // [kN] pivot row of step k
  int* used;      // [kN]
  double* red64;  // [8]
};

// No shared copy of the adjacency (it is re-read from global/L2 where needed):
// ~70 KB of shared memory and <= 64 registers let TWO instances share an SM.
size_t mtt_smem(int n) {
  return (size_t)kN * kN * 4 + (size_t)kN * 4 * 3 + (size_t)4 * kN * 4 + (size_t)kN * 8 + 64 + 256;
}

template <bool kMarg>
__global__ void __launch_bounds__(kThreads, 2) mtt_kernel(const float* __restrict__ adj_all, int n, int single,
                                                          double* __restrict__ logz, float* __restrict__ marg_all,
                                                          int32_t* __restrict__ status) {
  extern __shared__ __align__(16) char smraw[];
  MttSmem sm;
  {
    char* p = smraw;
    sm.inv = (float*)p; p += (size_t)kN * kN * 4;
    sm.shift = (float*)p; p += kN * 4;
    sm.diag = (float*)p; p += kN * 4;
    sm.rowmag = (float*)p; p += kN * 4;
    sm.rowbuf = (float*)p; p += 2 * kN * 4;
    sm.colbuf = (float*)p; p += 2 * kN * 4;
    sm.perm = (int*)p; p += kN * 4;
    sm.used = (int*)p; p += kN * 4;
    sm.red64 = (double*)p; p += 8 * 8;
  }
  __shared__ int flag_bad, flag_vac, piv_row;
  __shared__ double logdet;
  __shared__ int negs;

  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N1 = n + 1;
  const float* A = adj_all + (size_t)b * N1 * N1;
  if (tid == 0) { flag_bad = 0; flag_vac = 0; logdet = 0.0; negs = 0; }
  for (int e = tid; e < N1 * N1; e += kThreads)
    if (bad_input(__ldg(A + e))) flag_bad = 1;
  for (int e = tid; e < kN; e += kThreads) { sm.used[e] = 0; sm.rowmag[e] = 0.f; }
  __syncthreads();
  // column shifts and diagonal (spanning.py:90-120); thread d handles dependent d+1
  if (tid < n) {
    const int d = tid, dep = d + 1;
    float mx = ninf();
    for (int h = 0; h <= n; ++h)
      if (h != dep) mx = fmaxf(mx, __ldg(A + h * N1 + dep));
    if (mx == ninf()) flag_vac = 1;
    float s = 0.f;
    if (mx != ninf())
      for (int h = single ? 1 : 0; h <= n; ++h)
        if (h != dep) s += fexp(__ldg(A + h * N1 + dep) - mx);
    sm.shift[d] = mx;
    sm.diag[d] = s;
  }
  __syncthreads();
  if (flag_vac || flag_bad) {
    if (tid == 0) {
      status[b] = flag_bad ? SDB_ST_INVALID : SDB_ST_VACUOUS;
      logz[b] = ninfd();
    }
    if (kMarg)
      for (int e = tid; e < N1 * N1; e += kThreads) marg_all[(size_t)b * N1 * N1 + e] = 0.f;
    return;
  }
  // build the register block: rows r0..r0+3 (head h = r+1), cols c0..c0+7 (dep d = c+1)
  const int r0 = 4 * lane, c0 = 8 * warp;
  float a[4][8];
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    const int r = r0 + ii;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int c = c0 + jj;
      float v;
      if (r >= n || c >= n) {
        v = (r == c) ? 1.f : 0.f;  // identity padding
      } else if (single && r == 0) {
        v = fexp(__ldg(A + c + 1) - sm.shift[c]);  // row 0 <- root weights (Koo et al.)
      } else if (r == c) {
        v = sm.diag[c];
      } else {
        v = -fexp(__ldg(A + (r + 1) * N1 + c + 1) - sm.shift[c]);
      }
      a[ii][jj] = v;
    }
  }
  // original row magnitudes (numerics.py:143)
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    float mx = 0.f;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) mx = fmaxf(mx, fabsf(a[ii][jj]));
    atomicMax((int*)&sm.rowmag[r0 + ii], __float_as_int(mx));
  }
  __syncthreads();

  uint32_t usedm = 0;  // bit ii: row r0+ii has been a pivot row
  // ---- Gauss-Jordan with implicit partial pivoting
  bool singular = false;
  for (int k = 0; k < kN; ++k) {
    const int kb = k & 1;
    float* rowbuf = sm.rowbuf + kb * kN;
    float* colbuf = sm.colbuf + kb * kN;
    if (warp == (k >> 3)) {
      const int jj = k & 7;
      // argmax |a[r][k]| over unused rows r (first index on ties): |v| as float bits orders
      // like an unsigned int, so the warp argmax is two REDUX ops (max key, then the lowest
      // row holding it) instead of five shuffle rounds.  key = bits(|v|) + 1, 0 = no candidate.
      uint32_t bk = 0;
      int br = 0x7fffffff;
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) {
        const int r = r0 + ii;
        float v = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) if (q == jj) v = a[ii][q];
        colbuf[r] = v;
        const uint32_t key = ((usedm >> ii) & 1u) ? 0u : __float_as_uint(fabsf(v)) + 1u;
        if (key > bk) { bk = key; br = r; }  // rows ascending: strict '>' keeps the first
      }
      const uint32_t mk = __reduce_max_sync(0xffffffffu, bk);
      br = (int)__reduce_min_sync(0xffffffffu, (bk == mk) ? (uint32_t)br : 0x7fffffffu);
      if (lane == 0) {
        piv_row = br;
        sm.perm[k] = br;
      }
    }
    __syncthreads();
    const int p = piv_row;
    if ((p >> 2) == lane) usedm |= 1u << (p & 3);  // this lane's rows already pivoted (registers)
    // owners of row p publish it
    if ((p >> 2) == lane) {
      const int ii = p & 3;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q == ii) {
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) rowbuf[c0 + jj] = a[q][jj];
        }
    }
    __syncthreads();
    const float piv = rowbuf[k];
    // pivot bookkeeping (singularity test, sign, log|det|) happens after the loop, in
    // parallel over the recorded pivots: nothing fp64 on the per-step critical path
    if (tid == 0) sm.diag[k] = piv;  // diag is free once the Laplacian is in registers
    const float inv_piv = 1.f / piv;
    float cv[4];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) cv[ii] = colbuf[r0 + ii];
    float rv[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) rv[jj] = rowbuf[c0 + jj] * inv_piv;
    if (warp == (k >> 3)) {  // the warp owning column k (warp-uniform branch)
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) {
        const int r = r0 + ii;
        if (r == p) {
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) a[ii][jj] = (c0 + jj == k) ? inv_piv : rv[jj];
        } else {
          const float f = cv[ii];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) a[ii][jj] = (c0 + jj == k) ? -f * inv_piv : fmaf(-f, rv[jj], a[ii][jj]);
        }
      }
    } else {  // plain rank-1 update; the pivot row is overwritten by its owner lane
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) {
        const float f = cv[ii];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) a[ii][jj] = fmaf(-f, rv[jj], a[ii][jj]);
      }
      if ((p >> 2) == lane) {
#pragma unroll
        for (int ii = 0; ii < 4; ++ii)
          if (ii == (p & 3)) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) a[ii][jj] = rv[jj];
          }
      }
    }
  }
  (void)singular;
  __syncthreads();
  // log|det| = sum log|pivot| (numerics.py:157) in fp64, singular pivots
  // (numerics.py:143-146) and the pivot signs
  {
    double lg = 0.0;
    int neg = 0, sing = 0;
    if (tid < kN) {
      const float pv = sm.diag[tid];
      const float mag = fabsf(pv);
      sing = !(mag > 1e-12f * fmaxf(sm.rowmag[sm.perm[tid]], 1e-30f));
      lg = log((double)mag);
      neg = pv < 0.f;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lg += __shfl_xor_sync(0xffffffffu, lg, o);
    const int negc = __syncthreads_count(neg);
    if (__syncthreads_or(sing) && tid == 0) flag_vac = 1;
    if (lane == 0 && warp < kN / 32) sm.red64[warp] = lg;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w2 = 0; w2 < kN / 32; ++w2) t += sm.red64[w2];
      logdet = t;
      negs = negc;
    }
  }
  __syncthreads();
  // sign: pivot signs x permutation parity (numerics.py:149-155)
  if (tid == 0) {
    int parity = 0;
    // parity of k -> perm[k]: count transpositions via cycle decomposition
    for (int k = 0; k < kN; ++k) sm.used[k] = 0;
    for (int k = 0; k < kN; ++k) {
      if (sm.used[k]) continue;
      int len = 0, x = k;
      while (!sm.used[x]) { sm.used[x] = 1; x = sm.perm[x]; ++len; }
      parity ^= (len + 1) & 1;  // a cycle of length L has L-1 transpositions
    }
    const int sgn = ((negs + parity) & 1) ? -1 : 1;
    double ssum = 0.0;
    for (int d = 0; d < n; ++d) ssum += (double)sm.shift[d];
    const bool vac = flag_vac || sgn <= 0;
    flag_vac = vac;
    logz[b] = vac ? ninfd() : logdet + ssum;
    status[b] = vac ? SDB_ST_VACUOUS : SDB_ST_OK;
  }
  if (!kMarg) return;
  // q = inverse permutation (q[perm[k]] = k)
  __syncthreads();
  if (tid < kN) sm.used[sm.perm[tid]] = tid;  // reuse `used` as q
  __syncthreads();
  // A^{-1}[r][x] = M[p_r][q_x]  ->  M[i][j] goes to inv[q_i][p_j]
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    const int i = r0 + ii, qi = sm.used[i];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) sm.inv[sm.perm[c0 + jj] * kN + qi] = a[ii][jj];  // transposed: inv^T[x][d]
  }
  __syncthreads();
  float* mg = marg_all + (size_t)b * N1 * N1;
  const bool vac = flag_vac;
  // warp per head row h, lane over dependents: coalesced adjacency loads, and the transposed
  // inverse makes inv[d][h-1] for consecutive d contiguous (no bank conflicts)
  const float* invT = sm.inv;  // invT[x * kN + d] = A^{-1}[d][x]
  for (int h = warp; h < N1; h += kThreads / 32) {
    float av[5];
#pragma unroll
    for (int u = 0; u < 5; ++u) {
      const int dep = lane + 32 * u;
      av[u] = dep < N1 ? __ldg(A + (size_t)h * N1 + dep) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 5; ++u) {
      const int dep = lane + 32 * u;
      if (dep >= N1) continue;
      float v = 0.f;
      if (!vac && dep >= 1 && h != dep) {
        const int d = dep - 1;
        const float w = fexp(av[u] - sm.shift[d]);
        const float idd = invT[d * kN + d];
        if (single) {
          if (h == 0) v = w * invT[0 * kN + d];
          else v = w * ((d != 0 ? idd : 0.f) - ((h - 1) != 0 ? invT[(h - 1) * kN + d] : 0.f));
        } else {
          v = (h == 0) ? w * idd : w * (idd - invT[(h - 1) * kN + d]);
        }
        v = fminf(fmaxf(v, 0.f), 1.f);  // spanning.py:175
      }
      mg[(size_t)h * N1 + dep] = v;
    }
  }
}

int mtt_check(int64_t B, int n) {
  if (B < 0 || n < 1) return SDB_ERR_ARG;
  if (n > kN) return SDB_ERR_UNSUPPORTED;
  return SDB_OK;
}

}  // namespace

extern "C" int sdb_mtt(const float* adjacency, int64_t B, int32_t n, int32_t single_root, double* logz, float* marg,
                       int32_t* status, void* stream) {
  int rc = mtt_check(B, n);
  if (rc) return rc;
  if (!adjacency || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  const size_t smem = mtt_smem(n);
  cudaStream_t s = (cudaStream_t)stream;
  if (marg) {
    if (cudaFuncSetAttribute(mtt_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SDB_ERR_CUDA;
    mtt_kernel<true><<<(unsigned)B, kThreads, smem, s>>>(adjacency, n, single_root ? 1 : 0, logz, marg, status);
  } else {
    if (cudaFuncSetAttribute(mtt_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SDB_ERR_CUDA;
    mtt_kernel<false><<<(unsigned)B, kThreads, smem, s>>>(adjacency, n, single_root ? 1 : 0, logz, nullptr, status);
  }
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
