/* sdb200 -- C-ABI of the B200-native structured-inference kernels.
 *
 * Drop-in boundary for the hot path of the reference `structdist` 0.1.0
 * (/root/reference/pkg/src/structdist).  The reference has no FFI: its seam is
 * Python dispatch in dist.py (log_partition_info dist.py:68-84,
 * potential_marginals dist.py:96-117, marginals_info dist.py:120-129,
 * argmax_info dist.py:141-163) onto per-family functions.  Each export below
 * replaces one of those family functions, batched over a leading axis B.
 *
 * Conventions (every export):
 *   - all tensor pointers are DEVICE pointers, row-major, contiguous, with the
 *     reference's own axis order plus a leading batch axis; potentials fp32,
 *     integer structures int32, log-partitions fp64;
 *   - output pointers documented "nullable" may be NULL to skip that output
 *     (e.g. marginals == NULL runs the log-partition only);
 *   - `workspace` is caller-owned device scratch of at least the bytes the
 *     matching *_workspace() function returns (no allocation in hot calls);
 *   - `stream` is a cudaStream_t passed as void*; calls are stream-ordered and
 *     asynchronous, reentrant, and keep no mutable global state;
 *   - inputs are never written;
 *   - return value: SDB_OK or a negative SDB_ERR_* (argument / size / launch
 *     error).  Per-instance outcome goes to status[B] (SDB_ST_*).
 *
 * Status mapping onto the reference's exceptions (errors.py:4-24):
 *   SDB_ST_VACUOUS -> VacuousDistribution when marginals/argmax are asked
 *                     for (log_partition itself returns -inf, dist.py:68-87);
 *   SDB_ST_INVALID -> InvalidProblem (NaN / +inf potentials, numerics.py:25-28).
 */
#ifndef SDB200_H
#define SDB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDB_OK 0
#define SDB_ERR_ARG (-1)
#define SDB_ERR_WORKSPACE (-2)
#define SDB_ERR_CUDA (-3)
#define SDB_ERR_UNSUPPORTED (-4)

#define SDB_ST_OK 0
#define SDB_ST_VACUOUS 1
#define SDB_ST_INVALID 2

/* Library version (major*10000 + minor*100 + patch) and status strings. */
int sdb_version(void);
const char* sdb_status_string(int code);
/* CUDA runtime message of the last error an entry point returned SDB_ERR_CUDA for. */
const char* sdb_last_cuda_error(void);

/* ---------------------------------------------------------------- chain --
 * LinearChainCRF (chain.py:32-61): init [B,m], transitions [B,n-1,m,m]
 * indexed (step, prev, next).  n >= 1, 1 <= m <= 1024.
 *
 * sdb_chain_fb replaces chain._forward/_backward/forward_log_partition/
 * chain_marginals (chain.py:64-95): logz [B] (fp64), and, when non-NULL,
 * marg_init [B,m], marg_trans [B,n-1,m,m].
 */
size_t sdb_chain_fb_workspace(int64_t B, int32_t n, int32_t m);
int sdb_chain_fb(const float* init, const float* trans, int64_t B, int32_t n, int32_t m,
                 double* logz, float* marg_init, float* marg_trans, int32_t* status,
                 void* workspace, size_t ws_bytes, void* stream);

/* sdb_chain_viterbi replaces chain_argmax (chain.py:98-114): tags [B,n]
 * int32 (first-argmax ties, lowest tag index) and the best score [B] fp64. */
size_t sdb_chain_viterbi_workspace(int64_t B, int32_t n, int32_t m);
int sdb_chain_viterbi(const float* init, const float* trans, int64_t B, int32_t n, int32_t m,
                      int32_t* tags, double* score, int32_t* status,
                      void* workspace, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------ alignment --
 * MonotoneAlignmentCRF (alignment.py:30-59): theta [B,n+1,m+1,3] with moves
 * {0 DIAG from (i-1,j-1), 1 DOWN from (i-1,j), 2 RIGHT from (i,j-1)} scored
 * on arrival.  n >= 1, m >= 1 (m <= 351: strip kernels; larger m: an anti-diagonal
 * fp64 kernel, min(n, m) < 8192).
 *
 * sdb_nw_fb replaces _nw_forward/_nw_backward/nw_log_partition/nw_marginals
 * (alignment.py:62-118): logz [B]; marg [B,n+1,m+1,3] nullable.
 */
size_t sdb_nw_fb_workspace(int64_t B, int32_t n, int32_t m);
int sdb_nw_fb(const float* theta, int64_t B, int32_t n, int32_t m, double* logz, float* marg,
              int32_t* status, void* workspace, size_t ws_bytes, void* stream);

/* sdb_nw_viterbi replaces _nw_max_forward/_nw_walk/nw_argmax
 * (alignment.py:121-167): path [B,n+1,m+1] int8 = move index into each cell
 * on the best path (first maximum in DIAG, DOWN, RIGHT order), -1 elsewhere;
 * score [B] = best path score (fp64, max-plus). */
size_t sdb_nw_viterbi_workspace(int64_t B, int32_t n, int32_t m);
int sdb_nw_viterbi(const float* theta, int64_t B, int32_t n, int32_t m, int8_t* path, double* score,
                   int32_t* status, void* workspace, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------ CTC --
 * CTCDist (alignment.py:198-228): frame_potentials [B,T,V] (blank = 0),
 * targets [B,L] int32 in 1..V-1.  T >= 1, 2L+1 <= 1024.
 *
 * sdb_ctc_fb replaces _ctc_forward/_ctc_backward/ctc_log_partition/
 * ctc_marginals (alignment.py:248-301): logz [B]; marg [B,T,V] nullable
 * (state posteriors scatter-added by label).
 */
size_t sdb_ctc_fb_workspace(int64_t B, int32_t T, int32_t V, int32_t L);
int sdb_ctc_fb(const float* frame_potentials, const int32_t* targets, int64_t B, int32_t T, int32_t V,
               int32_t L, double* logz, float* marg, int32_t* status, void* workspace, size_t ws_bytes,
               void* stream);

/* sdb_ctc_viterbi replaces ctc_argmax/_ctc_walk (alignment.py:304-336):
 * labels [B,T] int32 = vocabulary id emitted per frame on the best expanded
 * path (predecessor ties s, s-1, s-2; final ties S-1, S-2); score [B]. */
size_t sdb_ctc_viterbi_workspace(int64_t B, int32_t T, int32_t V, int32_t L);
int sdb_ctc_viterbi(const float* frame_potentials, const int32_t* targets, int64_t B, int32_t T, int32_t V,
                    int32_t L, int32_t* labels, double* score, int32_t* status, void* workspace,
                    size_t ws_bytes, void* stream);

/* ------------------------------------------------------------- Tree-CRF --
 * TreeCRF (constituency.py:26-49): span_potentials [B,n,n,m] (i, j, label),
 * only i <= j read.  n >= 1: n <= 128 runs the shared-memory chart kernels,
 * larger n fp64 charts in global memory (workspace 3 x B n^2 doubles;
 * sdb_tree_viterbi allocates that scratch stream-ordered).
 *
 * sdb_tree_fb replaces _tree_charts/cky_log_partition/tree_marginals
 * (constituency.py:52-110): logz [B]; marg [B,n,n,m] nullable (0 for i > j
 * and unreachable spans).  Workspace: the label-folded span chart and the
 * per-span marginal multipliers, 2 x B n(n+1)/2 fp32. */
size_t sdb_tree_fb_workspace(int64_t B, int32_t n, int32_t m);
int sdb_tree_fb(const float* span_potentials, int64_t B, int32_t n, int32_t m, double* logz, float* marg,
                int32_t* status, void* workspace, size_t ws_bytes, void* stream);

/* sdb_tree_viterbi replaces cky_max_score/_tree_walk/tree_argmax
 * (constituency.py:72-133): labels [B,n,n] int32 = label of each span in the
 * best tree (first argmax label, first argmax split), -1 elsewhere. */
int sdb_tree_viterbi(const float* span_potentials, int64_t B, int32_t n, int32_t m, int32_t* labels,
                     double* score, int32_t* status, void* stream);

/* ---------------------------------------------------- Matrix-Tree (MTT) --
 * Directed non-projective SpanningTreeCRF (spanning.py:41-70):
 * adjacency [B,n+1,n+1] (head, dependent), node 0 = root, diagonal and
 * column 0 -inf.  1 <= n <= 128 (sdb_mtt_ex below: any n).  single_root != 0
 * selects the Koo et al.
 * single-root-edge Laplacian.
 *
 * sdb_mtt replaces _shifted_exp_weights/_build_laplacian/signed_log_det/
 * mtt_log_partition/mtt_marginals (spanning.py:90-175, numerics.py:128-159):
 * logz [B]; marg [B,n+1,n+1] nullable, clipped to [0,1].  No workspace. */
int sdb_mtt(const float* adjacency, int64_t B, int32_t n, int32_t single_root, double* logz, float* marg,
            int32_t* status, void* stream);

/* ------------------------------------------------ projective (Eisner) --
 * Directed projective SpanningTreeCRF: adjacency [B,n+1,n+1] (head, dep),
 * 1 <= n <= 128.
 *
 * sdb_eisner replaces _eisner_charts/eisner_log_partition/eisner_marginals
 * (spanning.py:183-280): logz [B]; marg [B,n+1,n+1] nullable, clipped.
 * sdb_kuhlmann replaces _reweight_root/kuhlmann_argmax (spanning.py:339-402),
 * the reference's public projective argmax: heads [B,n+1] int32 (heads[0] =
 * -1), best (reweighted) tabulation score [B]; bit-exact tie behaviour. */
int sdb_eisner(const float* adjacency, int64_t B, int32_t n, int32_t single_root, double* logz, float* marg,
               int32_t* status, void* stream);
int sdb_kuhlmann(const float* adjacency, int64_t B, int32_t n, int32_t single_root, int32_t* heads,
                 double* score, int32_t* status, void* stream);

/* ----------------------------------------------------------------- PCFG --
 * PCFG (constituency.py:184-243): root [B,NT], binary_rules [B,NT,S,S]
 * (S = NT+PT; children NTs then PTs), emissions [B,n,PT], sticky [B,n,n]
 * nullable ({0,-inf} span mask; NULL = all 0).  n <= 64, NT, PT <= 32.
 *
 * sdb_pcfg_fb replaces _pcfg_inside/pcfg_inside and the span-marginal part
 * of pcfg_gradients (constituency.py:246-340; marginals() returns only
 * {"sticky"}, dist.py:125-127): logz [B]; span_marg [B,n,n] nullable. */
size_t sdb_pcfg_fb_workspace(int64_t B, int32_t n, int32_t NT, int32_t PT);
int sdb_pcfg_fb(const float* root, const float* rules, const float* emissions, const float* sticky, int64_t B,
                int32_t n, int32_t NT, int32_t PT, double* logz, float* span_marg, int32_t* status,
                void* workspace, size_t ws_bytes, void* stream);

/* sdb_pcfg_grad replaces pcfg_gradients in full (constituency.py:292-340;
 * potential_marginals, dist.py:113-114): logz [B], span_marg [B,n,n] (the
 * "sticky" gradient), grad_root [B,NT], grad_rules [B,NT,S,S] (expected
 * anchored rule counts, may exceed 1), grad_emissions [B,n,PT]. */
size_t sdb_pcfg_grad_workspace(int64_t B, int32_t n, int32_t NT, int32_t PT);
int sdb_pcfg_grad(const float* root, const float* rules, const float* emissions, const float* sticky, int64_t B,
                  int32_t n, int32_t NT, int32_t PT, double* logz, float* span_marg, float* grad_root,
                  float* grad_rules, float* grad_emissions, int32_t* status, void* workspace, size_t ws_bytes,
                  void* stream);

/* sdb_pcfg_viterbi replaces pcfg_max_score, _pcfg_walk and pcfg_argmax
 * (constituency.py:275-277, 343-371): fp64 max-plus chart with the
 * reference's sums and first-maximum picks.  span_mask [B,n,n] int8 0/1,
 * score [B] = pcfg_max_score.  Workspace: the fp64 chart. */
size_t sdb_pcfg_viterbi_workspace(int64_t B, int32_t n, int32_t NT, int32_t PT);
int sdb_pcfg_viterbi(const float* root, const float* rules, const float* emissions, const float* sticky, int64_t B,
                     int32_t n, int32_t NT, int32_t PT, int8_t* span_mask, double* score, int32_t* status,
                     void* workspace, size_t ws_bytes, void* stream);

/* ----------------------------------------------------------- semi-Markov --
 * SemiMarkovCRF (chain.py:214-247): segment_potentials [B,n,s,m,m]
 * (start, width-1, prev label, label); virtual start label 0.
 *
 * sdb_semimarkov_fb replaces _sm_forward/_sm_backward/
 * semi_markov_log_partition/semi_markov_marginals (chain.py:250-298):
 * logz [B]; marg [B,n,s,m,m] nullable.  No workspace.
 * sdb_semimarkov_viterbi replaces semi_markov_argmax (chain.py:301-327):
 * segments [B,n,4] int32 rows (start, width, prev, label) in order,
 * num_segments [B], score [B]. */
int sdb_semimarkov_fb(const float* segment_potentials, int64_t B, int32_t n, int32_t s, int32_t m, double* logz,
                      float* marg, int32_t* status, void* stream);
size_t sdb_semimarkov_viterbi_workspace(int64_t B, int32_t n, int32_t s, int32_t m);
int sdb_semimarkov_viterbi(const float* segment_potentials, int64_t B, int32_t n, int32_t s, int32_t m,
                           int32_t* segments, int32_t* num_segments, double* score, int32_t* status,
                           void* workspace, size_t ws_bytes, void* stream);


/* ------------------------------------------------------------- sampling --
 * Exact samples (dist.py:179-212) with Gumbel-max picks (numerics.py:162-168).
 * `noise` [B, noise_per_instance] fp64 is the caller's Gumbel stream, drawn
 * from the reference's own Generator (np.random.default_rng(seed).gumbel),
 * consumed in the reference's pick order; num samples are drawn back to
 * back from it; used [B] reports the draws consumed.  fp64 log-semiring
 * charts in the workspace.  Stream bounds per sample: chain n*m; alignment
 * 3(n+m); CTC 2+3(T-1); Tree-CRF (2n-1)m + n^2; Eisner n + 4(n+1)^2.
 *
 * sdb_chain_sample: chain.py:117-129 (FFBS) -> tags [B,num,n].
 * sdb_nw_sample: alignment.py:121-150 -> path [B,num,n+1,m+1] (move or -1).
 * sdb_ctc_sample: alignment.py:304-318, 339-343 -> expanded-lattice state per
 *   frame [B,num,T].
 * sdb_tree_sample: constituency.py:113-140 -> labels [B,num,n,n] (-1 = no span).
 * sdb_eisner_decode: spanning.py:283-331: noise != NULL -> eisner_sample_arcs;
 *   noise == NULL -> eisner_max_arcs (max-plus charts, first-max picks).
 *   heads [B,num,n+1] (heads[0] = -1). */
size_t sdb_chain_sample_workspace(int64_t B, int32_t n, int32_t m);
int sdb_chain_sample(const float* init, const float* trans, int64_t B, int32_t n, int32_t m, const double* noise,
                     int64_t noise_per_instance, int32_t num, int32_t* tags, int32_t* used, int32_t* status,
                     void* workspace, size_t ws_bytes, void* stream);
size_t sdb_nw_sample_workspace(int64_t B, int32_t n, int32_t m);
int sdb_nw_sample(const float* theta, int64_t B, int32_t n, int32_t m, const double* noise,
                  int64_t noise_per_instance, int32_t num, int8_t* path, int32_t* used, int32_t* status,
                  void* workspace, size_t ws_bytes, void* stream);
size_t sdb_ctc_sample_workspace(int64_t B, int32_t T, int32_t V, int32_t L);
int sdb_ctc_sample(const float* frame_potentials, const int32_t* targets, int64_t B, int32_t T, int32_t V, int32_t L,
                   const double* noise, int64_t noise_per_instance, int32_t num, int32_t* states, int32_t* used,
                   int32_t* status, void* workspace, size_t ws_bytes, void* stream);
size_t sdb_tree_sample_workspace(int64_t B, int32_t n, int32_t m);
int sdb_tree_sample(const float* span_potentials, int64_t B, int32_t n, int32_t m, const double* noise,
                    int64_t noise_per_instance, int32_t num, int32_t* labels, int32_t* used, int32_t* status,
                    void* workspace, size_t ws_bytes, void* stream);
size_t sdb_eisner_decode_workspace(int64_t B, int32_t n);
int sdb_eisner_decode(const float* adjacency, int64_t B, int32_t n, int32_t single_root, const double* noise,
                      int64_t noise_per_instance, int32_t num, int32_t* heads, int32_t* used, int32_t* status,
                      void* workspace, size_t ws_bytes, void* stream);


/* sdb_cle replaces _find_cycle, _max_arborescence and cle_argmax
 * (spanning.py:410-509; single root via _reweight_root, spanning.py:339-350):
 * the non-projective argmax.  fp64 weights, the reference's tie rules ->
 * identical arcs.  heads [B,n+1] (heads[0] = -1); status VACUOUS when no
 * arborescence (or no single-root one) has finite score. */
size_t sdb_cle_workspace(int64_t B, int32_t n);
int sdb_cle(const float* adjacency, int64_t B, int32_t n, int32_t single_root, int32_t* heads, int32_t* status,
            void* workspace, size_t ws_bytes, void* stream);


/* Wilson's loop-erased random walk sampler (spanning.py:531-558), resumable:
 * sdb_wilson_begin puts the root (and root_child[b], nullable, for the
 * single-root variant after _condition_on_root_child) in the tree;
 * sdb_wilson_step consumes noise [B, cap] = the next cap draws of each
 * instance's Gumbel stream (n+1 per walk step), returning the cumulative
 * draws used [B] (int64) and status 0 done / 3 needs the next chunk / 4 step
 * cap exceeded (SamplerStepLimit).  parent [B, n+1] once done. */
size_t sdb_wilson_workspace(int64_t B, int32_t n);
int sdb_wilson_begin(int64_t B, int32_t n, const int32_t* root_child, int32_t* parent, int32_t* status,
                     void* workspace, size_t ws_bytes, void* stream);
int sdb_wilson_step(const float* adjacency, int64_t B, int32_t n, const double* noise, int64_t cap,
                    int64_t step_cap, int32_t* parent, int64_t* used, int32_t* status, void* workspace,
                    size_t ws_bytes, void* stream);


/* sdb_semimarkov_sample: semi_markov_sample (chain.py:330-344): segments
 * [B,num,n,4] (start, width, prev, label; last segment first), nseg
 * [B,num]; stream bound per sample n*s*m + m.
 * sdb_pcfg_sample: pcfg_sample (constituency.py:374-378): span_mask
 * [B,num,n,n]; stream bound per sample NT + S^2 n(n-1)/2; workspace as
 * sdb_pcfg_viterbi_workspace. */
size_t sdb_semimarkov_sample_workspace(int64_t B, int32_t n, int32_t s, int32_t m);
int sdb_semimarkov_sample(const float* segment_potentials, int64_t B, int32_t n, int32_t s, int32_t m,
                          const double* noise, int64_t noise_per_instance, int32_t num, int32_t* segments,
                          int32_t* nseg, int32_t* used, int32_t* status, void* workspace, size_t ws_bytes,
                          void* stream);
int sdb_pcfg_sample(const float* root, const float* rules, const float* emissions, const float* sticky, int64_t B,
                    int32_t n, int32_t NT, int32_t PT, const double* noise, int64_t noise_per_instance, int32_t num,
                    int8_t* span_mask, int32_t* used, int32_t* status, void* workspace, size_t ws_bytes,
                    void* stream);

/* ---- Matrix-Tree for any n ----------------------------------------------------
 * sdb_mtt serves n <= 128 (register-resident Laplacian, no workspace);
 * sdb_mtt_ex serves any n: n <= 128 forwards to sdb_mtt, larger n runs the
 * general fp64 Gauss-Jordan with the Laplacian and its inverse in the caller's
 * workspace (sdb_mtt_ex_workspace bytes; 0 for n <= 128).  Same outputs,
 * status codes and reference semantics as sdb_mtt (spanning.py:90-175). */
size_t sdb_mtt_ex_workspace(int64_t B, int32_t n);
int sdb_mtt_ex(const float* adjacency, int64_t B, int32_t n, int32_t single_root, double* logz, float* marg,
               int32_t* status, void* workspace, size_t ws_bytes, void* stream);

/* ---- ragged chain batches (per-instance lengths) -----------------------------
 * Replaces batch_map over chains of different lengths (dist.py:355-361) without
 * pad_chain (chain.py:161-176): init [B][m], trans [B][n-1][m][m] in the batch
 * layout, instance b uses its first lengths[b] positions (1 <= lengths[b] <= n);
 * marginals / tags past them are 0.  m <= 32 and n <= 193 (else
 * SDB_ERR_UNSUPPORTED: pad on the host instead).  Workspace as sdb_chain_fb. */
int sdb_chain_fb_lengths(const float* init, const float* trans, const int32_t* lengths, int64_t B, int32_t n,
                         int32_t m, double* logz, float* marg_init, float* marg_trans, int32_t* status,
                         void* workspace, size_t ws_bytes, void* stream);
int sdb_chain_viterbi_lengths(const float* init, const float* trans, const int32_t* lengths, int64_t B, int32_t n,
                              int32_t m, int32_t* tags, double* score, int32_t* status, void* stream);

/* ---- derived quantities: expected score under a potential tensor ------------
 * Replaces dist.py:306-347's host reduction _expected_score_under (masked_dot,
 * numerics.py:171-183) for cross_entropy / entropy / kl_divergence: out[b] +=
 * sum_e marg[b][e] * theta[b][e] over the parts with marg > 0 (0 * -inf = 0);
 * neginf[b] |= 1 when such a part has theta = -inf (supp p not in supp q -> the
 * cross-entropy is +inf).  Accumulates (zero out / neginf once for several
 * tensors).  marg, theta [B][len] fp32 device arrays. */
int sdb_masked_dot(const float* marg, const float* theta, int64_t B, int64_t len, double* out, int32_t* neginf,
                   void* stream);

/* ---- exact mode: float64 potentials in, float64 results out ----------------
 * The reference computes in float64 on float64 inputs; these entry points do
 * the same on the GPU (fp64 lattices / charts in the workspace, one CTA per
 * instance, the reference recurrences restated one-for-one) for callers that
 * compare at the reference's own tolerances.  Same layouts, statuses and
 * nullable-marginal convention as the fp32 entry points above; no size limits
 * beyond the workspace (alignment min(n, m) < 8192, CTC 2L+1 <= 12288,
 * MTT n <= 2048, Eisner n <= 4096).
 *   chain.py:64-95 / 250-298, alignment.py:62-118 / 248-301,
 *   constituency.py:52-110 / 246-340, spanning.py:90-175 / 183-280. */
size_t sdb_chain_fb_f64_workspace(int64_t B, int32_t n, int32_t m);
int sdb_chain_fb_f64(const double* init, const double* trans, int64_t B, int32_t n, int32_t m, double* logz,
                     double* marg_init, double* marg_trans, int32_t* status, void* workspace, size_t ws_bytes,
                     void* stream);
size_t sdb_semimarkov_fb_f64_workspace(int64_t B, int32_t n, int32_t s, int32_t m);
int sdb_semimarkov_fb_f64(const double* segment_potentials, int64_t B, int32_t n, int32_t s, int32_t m, double* logz,
                          double* marg, int32_t* status, void* workspace, size_t ws_bytes, void* stream);
size_t sdb_nw_fb_f64_workspace(int64_t B, int32_t n, int32_t m);
int sdb_nw_fb_f64(const double* theta, int64_t B, int32_t n, int32_t m, double* logz, double* marg, int32_t* status,
                  void* workspace, size_t ws_bytes, void* stream);
size_t sdb_ctc_fb_f64_workspace(int64_t B, int32_t T, int32_t V, int32_t L);
int sdb_ctc_fb_f64(const double* frame_potentials, const int32_t* targets, int64_t B, int32_t T, int32_t V,
                   int32_t L, double* logz, double* marg, int32_t* status, void* workspace, size_t ws_bytes,
                   void* stream);
size_t sdb_tree_fb_f64_workspace(int64_t B, int32_t n, int32_t m);
int sdb_tree_fb_f64(const double* span_potentials, int64_t B, int32_t n, int32_t m, double* logz, double* marg,
                    int32_t* status, void* workspace, size_t ws_bytes, void* stream);
/* span_marg NULL: log Z only; groot / grules / gemis non-NULL (with span_marg): pcfg_gradients too. */
size_t sdb_pcfg_f64_workspace(int64_t B, int32_t n, int32_t NT, int32_t PT, int32_t grad);
int sdb_pcfg_f64(const double* root, const double* rules, const double* emissions, const double* sticky, int64_t B,
                 int32_t n, int32_t NT, int32_t PT, double* logz, double* span_marg, double* groot, double* grules,
                 double* gemis, int32_t* status, void* workspace, size_t ws_bytes, void* stream);
/* pcfg_max_score / pcfg_argmax on float64 grammars (workspace: sdb_pcfg_viterbi_workspace). */
int sdb_pcfg_viterbi_f64(const double* root, const double* rules, const double* emissions, const double* sticky,
                         int64_t B, int32_t n, int32_t NT, int32_t PT, int8_t* span_mask, double* score,
                         int32_t* status, void* workspace, size_t ws_bytes, void* stream);
size_t sdb_mtt_f64_workspace(int64_t B, int32_t n);
int sdb_mtt_f64(const double* adjacency, int64_t B, int32_t n, int32_t single_root, double* logz, double* marg,
                int32_t* status, void* workspace, size_t ws_bytes, void* stream);
int sdb_eisner_f64(const double* adjacency, int64_t B, int32_t n, int32_t single_root, double* logz, double* marg,
                   int32_t* status, void* stream);
int sdb_masked_dot_f64(const double* marg, const double* theta, int64_t B, int64_t len, double* out,
                       int32_t* neginf, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SDB200_H */
