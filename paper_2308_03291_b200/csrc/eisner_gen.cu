// Projective (Eisner) spanning trees beyond the shared-memory chart kernels
// (n > 128): the reference's charts and chart-adjoint marginals
// (structdist spanning.py:183-280) in fp64 with all charts in global memory,
// one CTA (32 warps) per instance, one warp per span of the current width and
// one __syncthreads per width.
//
// Adjoint pass: within a width the only same-width targets of a span are its
// own il / ir adjoints (handled in order after a __syncwarp); every other
// target has a smaller width, and two spans of one width can hit the same
// smaller span, so those scatter-adds are fp64 atomics.
#include "common.cuh"

namespace {

constexpr int kT = 1024;
constexpr int kW = kT / 32;

struct WLse {
  double mx = ninfd(), s = 0.0;
  __device__ void add(double x) {
    if (x == ninfd()) return;
    if (x > mx) { s = s * exp(mx - x) + 1.0; mx = x; } else { s += exp(x - mx); }
  }
  __device__ double reduce() {
    double M = mx;
    for (int o = 16; o > 0; o >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
    if (M == ninfd()) return M;
    double t = (mx == ninfd()) ? 0.0 : s * exp(mx - M);
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    return M + log(t);
  }
};

template <typename TP, typename M>  // potential / marginal types (float64 = exact mode)
__global__ void __launch_bounds__(kT) eisner_gen_kernel(const TP* __restrict__ adj_all, int n, int single,
                                                        double* __restrict__ ws_all, double* __restrict__ logz,
                                                        M* __restrict__ marg_all, int32_t* __restrict__ status) {
  __shared__ int bad_s;
  __shared__ double z_s;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = n + 1;
  const size_t NN = (size_t)N * N;
  const TP* th = adj_all + (size_t)b * NN;
  double* cr = ws_all + (size_t)b * 8 * NN;
  double* cl = cr + NN;
  double* ir = cl + NN;
  double* il = ir + NN;
  double* bcr = il + NN;
  double* bcl = bcr + NN;
  double* bir = bcl + NN;
  double* bil = bir + NN;
  auto at = [&](int i, int j) { return (size_t)i * N + j; };
  auto T = [&](int h, int d) { return (double)__ldg(th + at(h, d)); };
  if (tid == 0) bad_s = 0;
  __syncthreads();
  {
    int bad = 0;
    for (size_t e = tid; e < NN; e += kT) {
      bad |= bad_value(__ldg(th + e));
      const bool diag = (e / N) == (e % N);
      cr[e] = diag ? 0.0 : ninfd();
      cl[e] = diag ? 0.0 : ninfd();
      ir[e] = ninfd();
      il[e] = ninfd();
      bcr[e] = bcl[e] = bir[e] = bil[e] = 0.0;
    }
    if (bad) bad_s = 1;
  }
  __syncthreads();
  // charts (spanning.py:183-207)
  for (int w = 1; w <= n; ++w) {
    for (int i = warp; i + w <= n; i += kW) {
      const int j = i + w;
      WLse f;
      for (int k = i + lane; k < j; k += 32) f.add(cr[at(i, k)] + cl[at(k + 1, j)]);
      const double fold = f.reduce();
      if (lane == 0) {
        ir[at(i, j)] = T(i, j) + fold;
        il[at(i, j)] = T(j, i) + fold;
      }
      __syncwarp();
      WLse r, l;
      for (int k = i + 1 + lane; k <= j; k += 32) r.add(ir[at(i, k)] + cr[at(k, j)]);
      for (int k = i + lane; k < j; k += 32) l.add(cl[at(i, k)] + il[at(k, j)]);
      const double vr = r.reduce(), vl = l.reduce();
      if (lane == 0) {
        cr[at(i, j)] = vr;
        cl[at(i, j)] = vl;
      }
    }
    __syncthreads();
  }
  // log Z (spanning.py:210-221)
  if (warp == 0) {
    double z;
    if (single) {
      WLse r;
      for (int c = 1 + lane; c <= n; c += 32) r.add(T(0, c) + cl[at(1, c)] + cr[at(c, n)]);
      z = r.reduce();
    } else {
      z = cr[at(0, n)];
    }
    if (lane == 0) {
      z_s = z;
      logz[b] = z;
      status[b] = bad_s ? SDB_ST_INVALID : (z == ninfd() ? SDB_ST_VACUOUS : SDB_ST_OK);
    }
  }
  __syncthreads();
  const double z = z_s;
  if (!marg_all || bad_s || z == ninfd()) return;  // marginals zeroed by the launcher
  M* mg = marg_all + (size_t)b * NN;
  // adjoints (spanning.py:224-280)
  if (single) {
    for (int c = 1 + tid; c <= n; c += kT) {
      const double t = T(0, c) + cl[at(1, c)] + cr[at(c, n)];
      const double p = t > ninfd() ? exp(t - z) : 0.0;
      mg[at(0, c)] = (M)fmin(fmax(p, 0.0), 1.0);
      bcl[at(1, c)] += p;
      bcr[at(c, n)] += p;
    }
  } else if (tid == 0) {
    bcr[at(0, n)] = 1.0;
  }
  __syncthreads();
  for (int w = n; w >= 1; --w) {
    for (int i = warp; i + w <= n; i += kW) {
      const int j = i + w;
      const size_t ij = at(i, j);
      {  // cl[i, j]
        const double bb = bcl[ij], c = cl[ij];
        if (bb > 0.0 && c > ninfd())
          for (int k = i + lane; k < j; k += 32) {
            const double wt = bb * exp(cl[at(i, k)] + il[at(k, j)] - c);
            atomicAdd(bcl + at(i, k), wt);
            atomicAdd(bil + at(k, j), wt);
          }
      }
      {  // cr[i, j]
        const double bb = bcr[ij], c = cr[ij];
        if (bb > 0.0 && c > ninfd())
          for (int k = i + 1 + lane; k <= j; k += 32) {
            const double wt = bb * exp(ir[at(i, k)] + cr[at(k, j)] - c);
            atomicAdd(bir + at(i, k), wt);
            atomicAdd(bcr + at(k, j), wt);
          }
      }
      __syncwarp();
      {  // il[i, j]: arc j -> i
        const double bb = bil[ij], c = il[ij];
        if (bb > 0.0 && c > ninfd()) {
          if (lane == 0) mg[at(j, i)] = (M)fmin(bb, 1.0);
          const double fold = c - T(j, i);
          for (int k = i + lane; k < j; k += 32) {
            const double wt = bb * exp(cr[at(i, k)] + cl[at(k + 1, j)] - fold);
            atomicAdd(bcr + at(i, k), wt);
            atomicAdd(bcl + at(k + 1, j), wt);
          }
        }
      }
      {  // ir[i, j]: arc i -> j
        const double bb = bir[ij], c = ir[ij];
        if (bb > 0.0 && c > ninfd()) {
          if (lane == 0) mg[ij] = (M)fmin(bb, 1.0);
          const double fold = c - T(i, j);
          for (int k = i + lane; k < j; k += 32) {
            const double wt = bb * exp(cr[at(i, k)] + cl[at(k + 1, j)] - fold);
            atomicAdd(bcr + at(i, k), wt);
            atomicAdd(bcl + at(k + 1, j), wt);
          }
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace

bool eisner_gen_ok(int n) { return n <= 4096; }

size_t eisner_gen_workspace(int64_t B, int n) { return (size_t)B * 8 * (n + 1) * (n + 1) * sizeof(double) + 256; }

// no workspace argument in sdb_eisner: stream-ordered scratch
template <typename TP, typename M>
int eisner_gen_launch_t(const TP* adj, int64_t B, int n, int single, double* logz, M* marg, int32_t* status,
                        cudaStream_t s) {
  if (!eisner_gen_ok(n)) return SDB_ERR_UNSUPPORTED;
  void* ws = nullptr;
  if (sdb_note(cudaMallocAsync(&ws, eisner_gen_workspace(B, n), s)) != cudaSuccess) return SDB_ERR_CUDA;
  if (marg && sdb_note(cudaMemsetAsync(marg, 0, (size_t)B * (n + 1) * (n + 1) * sizeof(M), s)) != cudaSuccess)
    return SDB_ERR_CUDA;
  eisner_gen_kernel<TP, M><<<(unsigned)B, kT, 0, s>>>(adj, n, single, (double*)ws, logz, marg, status);
  SDB_CHECK_LAUNCH();
  if (sdb_note(cudaFreeAsync(ws, s)) != cudaSuccess) return SDB_ERR_CUDA;
  return SDB_OK;
}

int eisner_gen_launch(const float* adj, int64_t B, int n, int single, double* logz, float* marg, int32_t* status,
                      cudaStream_t s) {
  return eisner_gen_launch_t<float, float>(adj, B, n, single, logz, marg, status, s);
}

// ---- exact mode (float64 adjacency and marginals)
extern "C" int sdb_eisner_f64(const double* adjacency, int64_t B, int32_t n, int32_t single_root, double* logz,
                              double* marg, int32_t* status, void* stream) {
  if (B < 0 || n < 1 || !adjacency || !logz || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  return eisner_gen_launch_t<double, double>(adjacency, B, n, single_root ? 1 : 0, logz, marg, status,
                                             (cudaStream_t)stream);
}
