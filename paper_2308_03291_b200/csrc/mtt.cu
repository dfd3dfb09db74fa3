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
// unused row p with max |a[p][k]| (a warp argmax inside the column's warp,
// two REDUX ops), publishes column k through shared memory (one CTA barrier
// per step), row p travels by shuffles inside each warp, and every thread does
// a register-blocked rank-1 update (32 FFMA; pivot-row scaling deferred).  Pivots
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
  int* prow;      // [2] pivot row of the step (double-buffered)
  float* colbuf;  // [2][kN]
  int* perm;      // [kN] pivot row of step k
  int* qinv;      // [kN] inverse pivot permutation
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
    sm.prow = (int*)p; p += 2 * kN * 4;
    sm.colbuf = (float*)p; p += 2 * kN * 4;
    sm.perm = (int*)p; p += kN * 4;
    sm.qinv = (int*)p; p += kN * 4;
    sm.red64 = (double*)p; p += 8 * 8;
  }
  __shared__ int flag_bad, flag_vac;

  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N1 = n + 1;
  const float* A = adj_all + (size_t)b * N1 * N1;
  if (tid == 0) { flag_bad = 0; flag_vac = 0; }
  for (int e = tid; e < N1 * N1; e += kThreads)
    if (bad_input(__ldg(A + e))) flag_bad = 1;
  for (int e = tid; e < kN; e += kThreads) sm.rowmag[e] = 0.f;
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
  // ---- Gauss-Jordan with implicit partial pivoting.  One CTA barrier per step: the warp
  // owning column k publishes the column and the pivot row index; the pivot row's entries
  // in a warp's own 8 columns live in one lane of that same warp, so they are broadcast
  // with shuffles instead of through shared memory.
  for (int k = 0; k < kN; ++k) {
    const int kb = k & 1;
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
        sm.prow[kb] = br;
        sm.perm[k] = br;
      }
    }
    __syncthreads();
    const int p = sm.prow[kb];
    const int pl = p >> 2, pi = p & 3;
    if (pl == lane) usedm |= 1u << pi;  // this lane's rows already pivoted (registers)
    const float piv = colbuf[p];
    // pivot bookkeeping (singularity test, sign, log|det|) happens after the loop, in
    // parallel over the recorded pivots: nothing fp64 on the per-step critical path
    if (tid == 0) sm.diag[k] = piv;  // diag is free once the Laplacian is in registers
    float inv_piv;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv_piv) : "f"(piv));
    // Lazy row scaling: the pivot row is NOT divided by the pivot here (multiplier 0 keeps it
    // as is); it stays piv_k x the true row, which later rank-1 updates preserve (they are
    // linear in the row), and the scatter below applies 1/piv_k once.  So every thread runs
    // the same 32 FFMA with no per-lane overwrite of the pivot row.
    float f[4];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) f[ii] = (r0 + ii == p) ? 0.f : colbuf[r0 + ii] * inv_piv;
    float rv[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const float x = pi == 0 ? a[0][jj] : pi == 1 ? a[1][jj] : pi == 2 ? a[2][jj] : a[3][jj];
      rv[jj] = __shfl_sync(0xffffffffu, x, pl);
    }
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) a[ii][jj] = fmaf(-f[ii], rv[jj], a[ii][jj]);
    if (warp == (k >> 3)) {  // column k: -a[r][k] / piv, and (scaled) 1 / piv on the pivot row
      const int jk = k & 7;
#pragma unroll
      for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int jj = 0; jj < 8; ++jj)
          if (jj == jk) a[ii][jj] = (r0 + ii == p) ? 1.f : -f[ii];
    }
  }
  __syncthreads();
  // log|det| = sum log|pivot| (numerics.py:157) in fp64, plus the column shifts; singular
  // pivots (numerics.py:143-146); sign = pivot signs x permutation parity (numerics.py:149-155),
  // the parity as the inversion count of k -> perm[k] mod 2 (all threads, no serial cycle walk)
  {
    double lg = 0.0;
    int neg = 0, sing = 0;
    if (tid < kN) {
      const float pv = sm.diag[tid];
      const float mag = fabsf(pv);
      sing = !(mag > 1e-12f * fmaxf(sm.rowmag[sm.perm[tid]], 1e-30f));
      lg = log((double)mag) + (tid < n ? (double)sm.shift[tid] : 0.0);
      neg = pv < 0.f;
    }
    int inv = 0;
    {
      const int i = tid & (kN - 1), j0 = (tid >> 7) * (kN / 4);
      const int pi = sm.perm[i];
#pragma unroll 8
      for (int j = j0; j < j0 + kN / 4; ++j) inv += (j > i) & (sm.perm[j] < pi);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lg += __shfl_xor_sync(0xffffffffu, lg, o);
    const int negc = __syncthreads_count(neg);
    const int par = __syncthreads_count(inv & 1);
    if (__syncthreads_or(sing) && tid == 0) flag_vac = 1;
    if (lane == 0 && warp < kN / 32) sm.red64[warp] = lg;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w2 = 0; w2 < kN / 32; ++w2) t += sm.red64[w2];
      const int sgn = ((negc + par) & 1) ? -1 : 1;
      const bool vac = flag_vac || sgn <= 0;
      flag_vac = vac;
      logz[b] = vac ? ninfd() : t;
      status[b] = vac ? SDB_ST_VACUOUS : SDB_ST_OK;
    }
  }
  if (!kMarg) return;
  // q = inverse permutation (q[perm[k]] = k)
  __syncthreads();
  if (tid < kN) sm.qinv[sm.perm[tid]] = tid;
  __syncthreads();
  // A^{-1}[r][x] = M[p_r][q_x]  ->  M[i][j] goes to inv[q_i][p_j]
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    const int i = r0 + ii, qi = sm.qinv[i];
    const float sc = 1.f / sm.diag[qi];  // the deferred pivot-row scaling
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) sm.inv[sm.perm[c0 + jj] * kN + qi] = a[ii][jj] * sc;  // transposed: inv^T[x][d]
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
