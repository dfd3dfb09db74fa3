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
// One CTA (512 threads = 16 warps) per instance, n <= 128 (padded to 128 with
// an identity block).  The 128x128 Laplacian lives in REGISTERS: warp w owns
// columns [8w, 8w+8), lane l owns rows [4l, 4l+4).
//
// Pipelined Gauss-Jordan (in-place inversion).  The 128 pivot steps are
// grouped in 16 panels of 8 = one warp's columns:
//   * producer: the warp owning panel b's columns runs its 8 pivot steps
//     alone (pivot row broadcast through a per-warp shared slot, rank-1
//     update of its 8 columns) and after EACH step publishes the pivot row
//     and multiplier column, signalled by a named-barrier ARRIVE (no wait);
//   * consumers: every other warp waits on that step's named barrier (SYNC)
//     and applies the rank-1 update to its own columns, one step behind the
//     producer -- the trailing updates overlap the producer's next steps.
// The next panel's warp starts producing as soon as it has applied the last
// step of the previous panel, so the critical path is the 128 producer steps
// (plus one consumer step per panel) and there is no CTA-wide barrier in the
// elimination.  Pivot rows are never divided in the loop (their multiplier is
// 0); the 1/pivot row scaling is applied once when the inverse is scattered.
// Pivoting: single root needs partial pivoting (row 0 holds the root
// weights; warp argmax by REDUX).  The multi-root Laplacian is column
// diagonally dominant (spanning.py:119), so partial pivoting picks the
// diagonal at every step and the pivot search is skipped (row k is the pivot
// of step k: static owner lane and register).
//
// Precision: with marginals the elimination runs in fp64 (fp32 elimination
// of the n=128 Laplacian leaves ~1e-6 absolute error in the marginals, which
// are differences of inverse entries); log Z alone runs the same kernel in
// fp32 (two CTAs per SM; pivots good to ~1e-7 relative, log|det| summed in fp64).
//
// Structural feasibility: before the elimination the CTA checks that a
// spanning arborescence with finite weight exists (bitset transitive closure
// of the finite arcs: every dependent reachable from the root; single root:
// from one root child).  An exactly singular Laplacian (a group of nodes cut
// off from the root) is thereby reported as vacuous (-inf) independent of
// rounding, as the reference's fp64 pivot test does (numerics.py:143-146).
#include "common.cuh"

namespace {

constexpr int kN = 128;
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kBitStride = 8;  // words per node row of the reachability bitsets (>= 5 for 129 nodes)

template <typename T>
struct MttSmem {
  T* inv;          // [kN*kN] A^{-1}, transposed (marginals only)
  T* F;            // [2][8][4][32] multiplier columns of a block, [step][row-in-lane][lane]
  T* slot;         // [kWarps][2][8] per-warp pivot-row broadcast slots (double-buffered)
  T* piv;          // [kN] pivot of step k
  T* diag;         // [kN] Laplacian diagonal
  T* rowmag;       // [kN] original row max-abs
  double* red64;   // [8]
  float* shift;    // [kN] column max s_d
  int* P;          // [2][8] pivot rows of a block
  int* perm;       // [kN] pivot row of step k
  int* qinv;       // [kN] inverse pivot permutation
  uint32_t* bits;  // [2][129][kBitStride] reachability bitsets
};

template <typename T, bool kMarg>
size_t mtt_smem() {
  return (kMarg ? (size_t)kN * kN * sizeof(T) : 0) + (size_t)2 * 8 * kN * sizeof(T) +
         (size_t)kWarps * 16 * sizeof(T) + (size_t)3 * kN * sizeof(T) + 64 + (size_t)kN * 4 + 64 +
         (size_t)2 * kN * 4 + (size_t)2 * 129 * kBitStride * 4 + 16 * 16;
}

template <typename T, bool kMarg>
__device__ __forceinline__ MttSmem<T> carve(char* p) {
  MttSmem<T> sm;
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 15) & ~(size_t)15;
    return r;
  };
  sm.inv = kMarg ? (T*)take((size_t)kN * kN * sizeof(T)) : nullptr;
  sm.F = (T*)take((size_t)2 * 8 * kN * sizeof(T));
  sm.slot = (T*)take((size_t)kWarps * 16 * sizeof(T));
  sm.piv = (T*)take(kN * sizeof(T));
  sm.diag = (T*)take(kN * sizeof(T));
  sm.rowmag = (T*)take(kN * sizeof(T));
  sm.red64 = (double*)take(64);
  sm.shift = (float*)take(kN * 4);
  sm.P = (int*)take(64);
  sm.perm = (int*)take(kN * 4);
  sm.qinv = (int*)take(kN * 4);
  sm.bits = (uint32_t*)take((size_t)2 * 129 * kBitStride * 4);
  return sm;
}

// order key of |v| (+1; 0 = no candidate): IEEE bits of a non-negative value order like integers
__device__ __forceinline__ uint64_t abs_key(double v) { return (uint64_t)__double_as_longlong(fabs(v)) + 1ull; }
__device__ __forceinline__ uint64_t abs_key(float v) { return (uint64_t)__float_as_uint(fabsf(v)) + 1ull; }
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t k) {
  const uint32_t hi = (uint32_t)(k >> 32);
  const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
  const uint32_t lo = (hi == mh) ? (uint32_t)k : 0u;
  const uint32_t ml = __reduce_max_sync(0xffffffffu, lo);
  return ((uint64_t)mh << 32) | ml;
}
__device__ __forceinline__ void atomic_max_abs(double* addr, double v) {  // v >= 0
  atomicMax((unsigned long long*)addr, (unsigned long long)__double_as_longlong(v));
}
__device__ __forceinline__ void atomic_max_abs(float* addr, float v) { atomicMax((int*)addr, __float_as_int(v)); }
__device__ __forceinline__ float to_f(double v) { return (float)v; }
// 1/x: MUFU seed + Newton steps (fp64: rcp.approx.ftz.f64 is ~2^-22, two steps reach fp64 rounding)
__device__ __forceinline__ double recip(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ float recip(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Does a spanning arborescence with finite weight exist?  R[i] (bits over the
// dependent index d = node - 1, built during the column-max pass) holds the
// finite arcs of node i plus i itself; repeated squaring closes it
// transitively.  Column 0 is -inf, so no path passes through the root and R[c]
// for c >= 1 only uses non-root arcs.  Multi-root: the root reaches every
// dependent.  Single root (spanning.py:116-117): some root child c with a
// finite root arc reaches every dependent.  CTA-uniform answer.
__device__ bool mtt_feasible(const float* __restrict__ A, int n, int single, uint32_t* bits, int* any_ok) {
  const int N1 = n + 1, NW = (n + 31) >> 5;
  const int tid = threadIdx.x;
  uint32_t* R0 = bits;
  uint32_t* R1 = bits + kBitStride * 129;
  auto full = [&](const uint32_t* r) {  // r covers every dependent d < n
    for (int w = 0; w < NW; ++w) {
      const uint32_t want = (n - 32 * w >= 32) ? 0xffffffffu : ((1u << (n - 32 * w)) - 1u);
      if ((r[w] & want) != want) return false;
    }
    return true;
  };
  if (tid == 0) *any_ok = 0;
  __syncthreads();
  // fast path (dense graphs): the root (multi-root) or one root child (single root) has a
  // finite arc to every other node
  if (!single) {
    if (tid == 0 && full(R0)) *any_ok = 1;
  } else if (tid >= 1 && tid < N1) {
    if (!is_ninf(__ldg(A + tid)) && full(R0 + tid * kBitStride)) *any_ok = 1;
  }
  if (__syncthreads_or(*any_ok != 0)) return true;
  for (int it = 0; (1 << it) < 2 * N1; ++it) {
    int changed = 0;
    if (tid < N1) {
      const uint32_t* cur = R0 + tid * kBitStride;
      uint32_t acc[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) acc[w] = w < NW ? cur[w] : 0u;
      if (!full(acc)) {
        for (int w = 0; w < NW; ++w) {
          uint32_t m = cur[w];
          while (m) {
            const int j = 32 * w + __ffs(m);  // node of dependent index 32 w + bit
            m &= m - 1;
            const uint32_t* rj = R0 + j * kBitStride;
#pragma unroll
            for (int w2 = 0; w2 < 4; ++w2) acc[w2] |= w2 < NW ? rj[w2] : 0u;
          }
        }
      }
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        if (w < NW) {
          changed |= acc[w] != cur[w];
          R1[tid * kBitStride + w] = acc[w];
        }
      }
    }
    const int any = __syncthreads_or(changed);
    uint32_t* t = R0;
    R0 = R1;
    R1 = t;
    if (!any) break;
  }
  if (!single) {
    if (tid == 0) *any_ok = full(R0);
  } else if (tid >= 1 && tid < N1) {
    if (!is_ninf(__ldg(A + tid)) && full(R0 + tid * kBitStride)) *any_ok = 1;
  }
  __syncthreads();
  return *any_ok != 0;
}

// the owner lane of pivot row p (= 4 lane + pi) copies its 8 entries to the warp's slot
template <typename T>
__device__ __forceinline__ void publish_row(const T (&a)[4][8], int pi, T* slot) {
  switch (pi) {  // warp-uniform
    case 0:
#pragma unroll
      for (int j = 0; j < 8; ++j) slot[j] = a[0][j];
      break;
    case 1:
#pragma unroll
      for (int j = 0; j < 8; ++j) slot[j] = a[1][j];
      break;
    case 2:
#pragma unroll
      for (int j = 0; j < 8; ++j) slot[j] = a[2][j];
      break;
    default:
#pragma unroll
      for (int j = 0; j < 8; ++j) slot[j] = a[3][j];
      break;
  }
}

template <typename T, bool kMarg, bool kPivot>
__global__ void __launch_bounds__(kThreads, sizeof(T) == 4 ? 2 : 1)
    mtt_kernel(const float* __restrict__ adj_all, int n, int single, double* __restrict__ logz,
               float* __restrict__ marg_all, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) char smraw[];
  const MttSmem<T> sm = carve<T, kMarg>(smraw);
  __shared__ int flag_bad, flag_vac, feas_ok;

  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N1 = n + 1;
  const float* A = adj_all + (size_t)b * N1 * N1;
  if (tid == 0) { flag_bad = 0; flag_vac = 0; }
  for (int e = tid; e < N1 * N1; e += kThreads)
    if (bad_input(__ldg(A + e))) flag_bad = 1;
  for (int e = tid; e < kN; e += kThreads) sm.rowmag[e] = T(0);
  __syncthreads();
  // column shifts and diagonal (spanning.py:90-120): the four thread quarters each scan a
  // quarter of the heads of dependent d+1 (coalesced rows) with an online max / sum, merged below
  {
    const int d = tid & (kN - 1), qtr = tid >> 7, dep = d + 1;
    const int hq = (N1 + 3) >> 2, h0 = qtr * hq, h1 = min(N1, h0 + hq);
    float* qm = (float*)sm.F;  // scratch: [4][kN] max, [4][kN] sum (F is free before the elimination)
    float* qs = qm + 4 * kN;
    // pass 1: column max over every head but the self-loop (spanning.py:93-95), and the
    // finite-arc bitsets of the feasibility check (a warp's lanes = 32 consecutive dependents)
    float mx = ninf();
    for (int h = h0; h < h1; ++h) {
      const float v = (d < n && h != dep) ? __ldg(A + h * N1 + dep) : ninf();
      mx = fmaxf(mx, v);
      const uint32_t word = __ballot_sync(0xffffffffu, d < n && (h == dep || !is_ninf(v)));
      if ((tid & 31) == 0) sm.bits[h * kBitStride + (d >> 5)] = word;
    }
    qm[qtr * kN + d] = mx;
    __syncthreads();
    float m = ninf();
#pragma unroll
    for (int q = 0; q < 4; ++q) m = fmaxf(m, qm[q * kN + d]);
    // pass 2: sum of exp over the heads that enter the diagonal (single root: not the root)
    float sum = 0.f;
    if (d < n && m != ninf())
      for (int h = max(h0, single); h < h1; ++h) sum += h == dep ? 0.f : fexp(__ldg(A + h * N1 + dep) - m);
    qs[qtr * kN + d] = sum;
    __syncthreads();
    if (tid < n) {
      if (m == ninf()) flag_vac = 1;
      sm.shift[tid] = m;
      sm.diag[tid] = (T)((qs[tid] + qs[kN + tid]) + (qs[2 * kN + tid] + qs[3 * kN + tid]));
    }
    __syncthreads();
  }
  if (!flag_vac && !flag_bad && !mtt_feasible(A, n, single, sm.bits, &feas_ok) && tid == 0)
    flag_vac = 1;  // exactly singular Laplacian
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
  T a[4][8];
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    const int r = r0 + ii;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int c = c0 + jj;
      T v;
      if (r >= n || c >= n) {
        v = (r == c) ? T(1) : T(0);  // identity padding
      } else if (single && r == 0) {
        v = (T)fexp(__ldg(A + c + 1) - sm.shift[c]);  // row 0 <- root weights (Koo et al.)
      } else if (r == c) {
        v = sm.diag[c];
      } else {
        v = -(T)fexp(__ldg(A + (r + 1) * N1 + c + 1) - sm.shift[c]);
      }
      a[ii][jj] = v;
    }
  }
  // original row magnitudes (numerics.py:143)
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    T mx = T(0);
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) mx = fmax(mx, fabs(a[ii][jj]));
    atomic_max_abs(&sm.rowmag[r0 + ii], mx);
  }

  uint32_t usedm = 0;  // bit ii: row r0+ii has been a pivot row
  T* myslot = sm.slot + warp * 16;
  __syncthreads();  // rowmag complete; the shift scratch in F is dead
  for (int blk = 0; blk < kN / 8; ++blk) {
    const int buf = blk & 1;
    T* Fb = sm.F + buf * 8 * kN;
    int* Pb = sm.P + buf * 8;
    if (warp == blk) {
      // ---- producer: 8 pivot steps on this warp's own columns (unrolled: column kk is static)
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        int p, pl, pi;
        if constexpr (kPivot) {
          // argmax |a[r][kk]| over unused rows (first index on ties; numerics.py:140-142)
          uint64_t bk = 0;
          int br = 0x7fffffff;
#pragma unroll
          for (int ii = 0; ii < 4; ++ii) {
            const uint64_t key = ((usedm >> ii) & 1u) ? 0ull : abs_key(a[ii][kk]);
            if (key > bk) { bk = key; br = r0 + ii; }  // rows ascending: strict '>' keeps the first
          }
          const uint64_t mk = warp_max_u64(bk);
          p = (int)__reduce_min_sync(0xffffffffu, (bk == mk) ? (uint32_t)br : 0x7fffffffu);
          pl = p >> 2;
          pi = p & 3;
        } else {
          p = 8 * blk + kk;
          pl = p >> 2;
          pi = kk & 3;  // static
        }
        T* s = myslot + (kk & 1) * 8;
        if (lane == pl) {
          usedm |= 1u << pi;
          publish_row(a, pi, s);
        }
        __syncwarp();
        T rv[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) rv[jj] = s[jj];
        const T piv = rv[kk], ip = recip(piv);
        T f[4];
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) f[ii] = (r0 + ii == p) ? T(0) : a[ii][kk] * ip;
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) Fb[(kk * 4 + ii) * 32 + lane] = f[ii];
        if (lane == 0) {
          Pb[kk] = p;
          sm.perm[8 * blk + kk] = p;
          sm.piv[8 * blk + kk] = piv;
        }
        // publish step kk to the consumers (release; they SYNC on the same named barrier)
        asm volatile("bar.arrive %0, %1;" ::"r"(1 + kk), "r"(kThreads) : "memory");
        // the next column first: the next step's pivot search waits only on it
        if (kk < 7) {
#pragma unroll
          for (int ii = 0; ii < 4; ++ii) a[ii][kk + 1] = fma(-f[ii], rv[kk + 1], a[ii][kk + 1]);
        }
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            if (jj != kk && jj != kk + 1) a[ii][jj] = fma(-f[ii], rv[jj], a[ii][jj]);
          a[ii][kk] = (r0 + ii == p) ? T(1) : -f[ii];  // column kk of the (row-scaled) inverse
        }
      }
    } else {
      // ---- consumer: apply the panel's rank-1 updates to this warp's columns, step by step
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + kk), "r"(kThreads) : "memory");
        int p, pl, pi;
        if constexpr (kPivot) {
          p = Pb[kk];
          pi = p & 3;
        } else {
          p = 8 * blk + kk;
          pi = kk & 3;
        }
        pl = p >> 2;
        T* s = myslot + (kk & 1) * 8;
        if (lane == pl) {
          usedm |= 1u << pi;
          publish_row(a, pi, s);
        }
        __syncwarp();
        T rv[8], f[4];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) rv[jj] = s[jj];
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) f[ii] = Fb[(kk * 4 + ii) * 32 + lane];
#pragma unroll
        for (int ii = 0; ii < 4; ++ii)
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) a[ii][jj] = fma(-f[ii], rv[jj], a[ii][jj]);
      }
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
      const T pv = sm.piv[tid];
      const T mag = fabs(pv);
      sing = !(mag > T(1e-12) * fmax(sm.rowmag[sm.perm[tid]], T(1e-30)));
      lg = log((double)mag) + (tid < n ? (double)sm.shift[tid] : 0.0);
      neg = pv < T(0);
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
  if constexpr (kMarg) {
    // q = inverse permutation (q[perm[k]] = k)
    __syncthreads();
    if (tid < kN) sm.qinv[sm.perm[tid]] = tid;
    __syncthreads();
    // A^{-1}[r][x] = M[p_r][q_x]  ->  M[i][j] goes to inv[q_i][p_j]
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const int i = r0 + ii, qi = sm.qinv[i];
      const T sc = T(1) / sm.piv[qi];  // the deferred pivot-row scaling
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) sm.inv[sm.perm[c0 + jj] * kN + qi] = a[ii][jj] * sc;  // inv^T[x][d]
    }
    __syncthreads();
    float* mg = marg_all + (size_t)b * N1 * N1;
    const bool vac = flag_vac;
    // warp per head row h, lane over dependents: coalesced adjacency loads, and the transposed
    // inverse makes inv[d][h-1] for consecutive d contiguous
    const T* invT = sm.inv;  // invT[x * kN + d] = A^{-1}[d][x]
    for (int h = warp; h < N1; h += kWarps) {
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
        T v = T(0);
        if (!vac && dep >= 1 && h != dep) {
          const int d = dep - 1;
          const T w = (T)fexp(av[u] - sm.shift[d]);
          const T idd = invT[d * kN + d];
          if (single) {
            if (h == 0) v = w * invT[0 * kN + d];
            else v = w * ((d != 0 ? idd : T(0)) - ((h - 1) != 0 ? invT[(h - 1) * kN + d] : T(0)));
          } else {
            v = (h == 0) ? w * idd : w * (idd - invT[(h - 1) * kN + d]);
          }
          v = fmin(fmax(v, T(0)), T(1));  // spanning.py:175
        }
        mg[(size_t)h * N1 + dep] = to_f(v);
      }
    }
  }
}

}  // namespace

size_t mtt_gen_workspace(int64_t B, int n);
int mtt_gen_launch(const float* adjacency, int64_t B, int n, int single, double* logz, float* marg, int32_t* status,
                   void* workspace, size_t ws_bytes, cudaStream_t s);

namespace {

int mtt_check(int64_t B, int n) {
  if (B < 0 || n < 1) return SDB_ERR_ARG;
  if (n > kN) return SDB_ERR_UNSUPPORTED;
  return SDB_OK;
}

template <typename T, bool kMarg, bool kPivot>
int launch_mtt(const float* adjacency, int64_t B, int n, int sr, double* logz, float* marg, int32_t* status,
               cudaStream_t s) {
  const size_t smem = mtt_smem<T, kMarg>();
  if (sdb_set_smem((const void*)mtt_kernel<T, kMarg, kPivot>, smem) != cudaSuccess)
    return SDB_ERR_CUDA;
  mtt_kernel<T, kMarg, kPivot><<<(unsigned)B, kThreads, smem, s>>>(adjacency, n, sr, logz, marg, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

}  // namespace

extern "C" int sdb_mtt(const float* adjacency, int64_t B, int32_t n, int32_t single_root, double* logz, float* marg,
                       int32_t* status, void* stream) {
  int rc = mtt_check(B, n);
  if (rc) return rc;
  if (!adjacency || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int sr = single_root ? 1 : 0;
  // log Z alone needs only the pivots (fp32 elimination, two CTAs per SM); the marginals
  // (differences of inverse entries) need the fp64 elimination
  // (single root pivots; the column diagonally dominant multi-root Laplacian does not need to)
  if (marg)
    return sr ? launch_mtt<double, true, true>(adjacency, B, n, sr, logz, marg, status, s)
              : launch_mtt<double, true, false>(adjacency, B, n, sr, logz, marg, status, s);
  return sr ? launch_mtt<float, false, true>(adjacency, B, n, sr, logz, nullptr, status, s)
            : launch_mtt<float, false, false>(adjacency, B, n, sr, logz, nullptr, status, s);
}

// n > 128 (or any n): the general fp64 kernel (mtt_gen.cu) with a caller workspace;
// n <= 128 takes the register-resident kernel and needs no workspace.
extern "C" size_t sdb_mtt_ex_workspace(int64_t B, int32_t n) { return n <= kN ? 0 : mtt_gen_workspace(B, n); }

extern "C" int sdb_mtt_ex(const float* adjacency, int64_t B, int32_t n, int32_t single_root, double* logz, float* marg,
                          int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  if (B < 0 || n < 1 || !adjacency || !logz || !status) return SDB_ERR_ARG;
  if (n <= kN) return sdb_mtt(adjacency, B, n, single_root, logz, marg, status, stream);
  if (B == 0) return SDB_OK;
  return mtt_gen_launch(adjacency, B, n, single_root ? 1 : 0, logz, marg, status, workspace, ws_bytes,
                        (cudaStream_t)stream);
}
