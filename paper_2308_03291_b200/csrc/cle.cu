// Non-projective argmax: maximum arborescence by greedy best incoming edges
// plus cycle contraction (Chu-Liu-Edmonds), with the single-root constraint
// enforced by root reweighting.
//
// Reference: spanning.py:410-509 (_find_cycle, _max_arborescence,
// cle_argmax) and 339-350 (_reweight_root).  The reference recurses on the
// contracted weight matrix; here the recursion is a loop over contraction
// levels in ONE CTA per instance: the O(S^2) parts (best heads, the
// contracted matrix, entering / leaving edges) are parallel over nodes, the
// O(S) parts (cycle search, id maps, expansion) run on thread 0.  All
// weights are fp64 with the reference's arithmetic (adjusted = w[u,v] -
// w[best_head[v], v]) and tie rules (np.argmax first maximum, strict '>' in
// cycle order), so the arcs are bit-identical.
//
// Workspace per instance: two (n+1)^2 fp64 weight buffers + per-level records
// (size, keep, best heads, cycle, enter/leave) as (n+1)^2 int32 arrays.
#include "common.cuh"

namespace {

constexpr int kT = 256;

struct CleWs {
  double* W;   // [B][2][N][N]
  int* rec;    // [B][5][N][N]: keep, bh, cyc, enter, leave (level-major)
  int* meta;   // [B][2][N]: size per level, cycle length per level
};

__global__ void __launch_bounds__(kT) cle_kernel(const float* __restrict__ adj_all, int n, int single, CleWs ws,
                                                 int32_t* __restrict__ heads_all, int32_t* __restrict__ status) {
  const int b = blockIdx.x, tid = threadIdx.x;
  const int N = n + 1;
  const float* adj = adj_all + (size_t)b * N * N;
  double* Wa = ws.W + (size_t)b * 2 * N * N;
  double* Wb = Wa + (size_t)N * N;
  int* KEEP = ws.rec + (size_t)b * 5 * N * N;
  int* BH = KEEP + (size_t)N * N;
  int* CYC = BH + (size_t)N * N;
  int* ENT = CYC + (size_t)N * N;
  int* LEA = ENT + (size_t)N * N;
  int* SZ = ws.meta + (size_t)b * 2 * N;
  int* CL = SZ + N;
  int32_t* heads = heads_all + (size_t)b * N;
  __shared__ int flag_bad, flag_vac, ncyc, top_level, new_id[1024], parent[1024], par2[1024];
  __shared__ double rw_c;
  if (tid == 0) {
    flag_bad = 0;
    flag_vac = 0;
  }
  __syncthreads();
  // inputs + root reweighting constant (spanning.py:339-350)
  {
    int bad = 0;
    double lo = 1e300, hi = -1e300;
    int fin = 0;
    for (int e = tid; e < N * N; e += kT) {
      const float x = adj[e];
      const int h = e / N, d = e - h * N;
      if (h != d && d != 0) bad |= bad_input(x);
      if (x != ninf() && x == x && x != __int_as_float(0x7f800000)) {
        lo = fmin(lo, (double)x);
        hi = fmax(hi, (double)x);
        fin = 1;
      }
    }
    __shared__ double lo_s[kT / 32], hi_s[kT / 32];
    __shared__ int fin_s[kT / 32];
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      fin |= __shfl_xor_sync(0xffffffffu, fin, o);
    }
    if ((tid & 31) == 0) {
      lo_s[tid >> 5] = lo;
      hi_s[tid >> 5] = hi;
      fin_s[tid >> 5] = fin;
    }
    if (bad) atomicOr(&flag_bad, 1);
    __syncthreads();
    if (tid == 0) {
      double L = lo_s[0], H = hi_s[0];
      int F = fin_s[0];
      for (int q = 1; q < kT / 32; ++q) {
        L = fmin(L, lo_s[q]);
        H = fmax(H, hi_s[q]);
        F |= fin_s[q];
      }
      rw_c = (double)n * (H - L) + 1.0;
      if (single && !F) flag_vac = 1;
    }
    __syncthreads();
  }
  if (flag_bad || flag_vac) {
    if (tid == 0) status[b] = flag_bad ? SDB_ST_INVALID : SDB_ST_VACUOUS;
    for (int e = tid; e < N; e += kT) heads[e] = -1;
    return;
  }
  for (int e = tid; e < N * N; e += kT) {
    double v = (double)adj[e];
    if (single && e >= 1 && e < N) v = v - rw_c;  // root row, dependents 1..n
    Wa[e] = v;
  }
  __syncthreads();
  int S = N, level = 0;
  double* W = Wa;
  double* Wn = Wb;
  while (true) {
    if (tid == 0) SZ[level] = S;
    int* bh = BH + (size_t)level * N;
    // best incoming edge per dependent: first maximum of the column with the
    // self entry masked (spanning.py:443-449)
    for (int v = 1 + tid; v < S; v += kT) {
      double best = ninfd();
      int h = 0;
      for (int u = 0; u < S; ++u) {
        const double x = (u == v) ? ninfd() : W[(size_t)u * S + v];
        if (x > best) {
          best = x;
          h = u;
        }
      }
      bh[v] = h;
      if (best == ninfd()) atomicOr(&flag_vac, 1);
    }
    __syncthreads();
    if (flag_vac) break;
    int* cyc = CYC + (size_t)level * N;
    if (tid == 0) {
      // _find_cycle (spanning.py:410-425): lowest start, walk to a resolved
      // node or back into the current path
      int len = 0;
      for (int x = 0; x < S; ++x) new_id[x] = 0;  // 0 = unseen, 1 = resolved, 2 = on path
      new_id[0] = 1;
      for (int start = 1; start < S && len == 0; ++start) {
        if (new_id[start] == 1) continue;
        int plen = 0, node = start;
        while (new_id[node] == 0) {
          new_id[node] = 2;
          par2[node] = plen;  // position in path
          parent[plen++] = node;
          node = bh[node];
        }
        if (new_id[node] == 2) {
          for (int q = par2[node]; q < plen; ++q) cyc[len++] = parent[q];
        }
        for (int q = 0; q < plen; ++q) new_id[parent[q]] = 1;
      }
      ncyc = len;
      CL[level] = len;
    }
    __syncthreads();
    if (ncyc == 0) break;
    // contraction (spanning.py:455-485): keep = non-cycle nodes in order, c* last
    int* keep = KEEP + (size_t)level * N;
    if (tid == 0) {
      for (int x = 0; x < S; ++x) par2[x] = 0;
      for (int q = 0; q < ncyc; ++q) par2[cyc[q]] = 1;
      int c = 0;
      for (int x = 0; x < S; ++x)
        if (!par2[x]) {
          new_id[x] = c;
          keep[c++] = x;
        }
      top_level = c;  // c* = number of kept nodes
    }
    __syncthreads();
    const int cs = top_level, S2 = cs + 1;
    int* ent = ENT + (size_t)level * N;
    int* lea = LEA + (size_t)level * N;
    for (int nu = tid; nu < cs; nu += kT) {
      const int u = keep[nu];
      for (int nv = 0; nv < cs; ++nv) {
        const int v = keep[nv];
        Wn[(size_t)nu * S2 + nv] = (u != v) ? W[(size_t)u * S + v] : ninfd();
      }
      double best = ninfd();
      int arg = -1;
      for (int q = 0; q < ncyc; ++q) {
        const int v = cyc[q];
        const double w = W[(size_t)u * S + v];
        if (w == ninfd()) continue;
        const double adjd = w - W[(size_t)bh[v] * S + v];
        if (adjd > best) {
          best = adjd;
          arg = v;
        }
      }
      Wn[(size_t)nu * S2 + cs] = (arg >= 0) ? best : ninfd();
      ent[nu] = arg;
      best = ninfd();
      arg = -1;
      if (u != 0) {
        for (int q = 0; q < ncyc; ++q) {
          const int v = cyc[q];
          const double w = W[(size_t)v * S + u];
          if (w > best) {
            best = w;
            arg = v;
          }
        }
      }
      Wn[(size_t)cs * S2 + nu] = (arg >= 0) ? best : ninfd();
      lea[nu] = arg;
    }
    if (tid == 0) Wn[(size_t)cs * S2 + cs] = ninfd();
    __syncthreads();
    double* t = W;
    W = Wn;
    Wn = t;
    S = S2;
    ++level;
  }
  if (flag_vac) {
    if (tid == 0) status[b] = SDB_ST_VACUOUS;
    for (int e = tid; e < N; e += kT) heads[e] = -1;
    return;
  }
  if (tid != 0) return;
  // expansion (spanning.py:487-499), deepest level first
  const int deep = level;
  for (int v = 1; v < SZ[deep]; ++v) parent[v] = BH[(size_t)deep * N + v];
  for (int lv = deep - 1; lv >= 0; --lv) {
    const int Sl = SZ[lv], cs = SZ[lv + 1] - 1;
    const int* keep = KEEP + (size_t)lv * N;
    const int* ent = ENT + (size_t)lv * N;
    const int* lea = LEA + (size_t)lv * N;
    const int* bh = BH + (size_t)lv * N;
    const int* cyc = CYC + (size_t)lv * N;
    for (int x = 0; x < Sl; ++x) par2[x] = -1;
    int entry = -1;
    for (int nd = 1; nd <= cs; ++nd) {
      const int nh = parent[nd];
      if (nd == cs) {
        entry = ent[nh];
        par2[entry] = keep[nh];
      } else if (nh == cs) {
        par2[keep[nd]] = lea[nd];
      } else {
        par2[keep[nd]] = keep[nh];
      }
    }
    for (int q = 0; q < CL[lv]; ++q)
      if (cyc[q] != entry) par2[cyc[q]] = bh[cyc[q]];
    for (int x = 0; x < Sl; ++x) parent[x] = par2[x];
  }
  heads[0] = -1;
  int roots = 0;
  for (int d = 1; d < N; ++d) {
    heads[d] = parent[d];
    roots += parent[d] == 0;
  }
  // cle_argmax (spanning.py:505-508): the reweighting must leave one root edge
  status[b] = (single && roots != 1) ? SDB_ST_VACUOUS : SDB_ST_OK;
}

CleWs cle_carve(void* base, int64_t B, int n, size_t* bytes) {
  const size_t N = n + 1;
  Carve c(base);
  CleWs w;
  w.W = c.take<double>((size_t)B * 2 * N * N);
  w.rec = c.take<int>((size_t)B * 5 * N * N);
  w.meta = c.take<int>((size_t)B * 2 * N);
  *bytes = c.used;
  return w;
}

}  // namespace

extern "C" size_t sdb_cle_workspace(int64_t B, int32_t n) {
  size_t bytes = 0;
  cle_carve(nullptr, B, n, &bytes);
  return bytes;
}

extern "C" int sdb_cle(const float* adjacency, int64_t B, int32_t n, int32_t single_root, int32_t* heads,
                       int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  if (B < 0 || n < 1) return SDB_ERR_ARG;
  if (n > 1023) return SDB_ERR_UNSUPPORTED;
  if (!adjacency || !heads || !status) return SDB_ERR_ARG;
  if (B == 0) return SDB_OK;
  size_t need = 0;
  CleWs ws = cle_carve(workspace, B, n, &need);
  if (!workspace || ws_bytes < need) return SDB_ERR_WORKSPACE;
  cle_kernel<<<(unsigned)B, kT, 0, (cudaStream_t)stream>>>(adjacency, n, single_root, ws, heads, status);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}
