/*
 * specexec_b200.h -- C ABI of the B200-native SpecExec hot path.
 *
 * The reference (`speckit`, pure Python + numpy) has no native boundary: its
 * hot path is the Python call chain
 *   generate_specexec  pkg/src/speckit/engine.py:92-131
 *     precompute       pkg/src/speckit/engine.py:73-89
 *       build_sssp     pkg/src/speckit/tree.py:240-327
 *       LanguageModel.next_distributions  pkg/src/speckit/models.py:47-52
 *     apply_warp/sample pkg/src/speckit/sampling.py:66-113
 * The entry points below are what a ctypes binding of that chain calls (see
 * INTEGRATION.md). Each one names the reference interface whose semantics it
 * implements.
 *
 * Conventions
 *  - Device buffers are allocated by the caller (PyTorch) and passed as raw
 *    pointers plus explicit sizes; kernels never allocate or free.
 *  - Every call is asynchronous on the given stream (cudaStream_t; NULL = the
 *    legacy default stream) unless documented otherwise.
 *  - Return: 0 ok; < 0 argument error (the Python layer raises ValueError);
 *    > 0 a cudaError_t (RuntimeError). sx_last_error() returns a thread-local
 *    message for the last failure on the calling thread.
 *  - No global mutable state besides the thread-local error string and an
 *    internal cache of TMA descriptors (mutex-protected).
 */
#ifndef SPECEXEC_B200_H_
#define SPECEXEC_B200_H_

#include <stdint.h>
#include <cuda_runtime.h>

#if defined(__GNUC__)
#define SX_API __attribute__((visibility("default")))
#else
#define SX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- misc */
SX_API int sx_abi_version(void);
SX_API const char* sx_last_error(void);
/* number of kernels launched through this library since it was loaded */
SX_API long long sx_launch_count(void);

/* ----------------------------------------------- KG: dense projections
 * Y[t, f] (op)= sum_k X[t, k] * W[f, k]; bf16 in, fp32 accumulate on tcgen05.
 * Replaces the dense part of LanguageModel.next_distributions
 * (pkg/src/speckit/models.py:47-52) for Llama-shaped models.
 *   W   [N, K] bf16 row-major (nn.Linear weight layout)
 *   W2  optional second weight [N, K] (SwiGLU up-projection) or NULL
 *   X   [M, K] bf16 row-major, contiguous
 *   out [M, ldo] bf16 or fp32 depending on the epilogue
 *   ws  fp32 split-K workspace (sx_gemm_plan reports the size), may be NULL
 *       when no split is needed. splits_req <= 0 picks automatically.
 */
enum {
  SX_EPI_BF16 = 0,        /* out bf16  = acc                       */
  SX_EPI_F32 = 1,         /* out fp32  = acc                       */
  SX_EPI_ADD_F32 = 2,     /* out fp32 += acc (residual stream)     */
  SX_EPI_SWIGLU_BF16 = 3, /* out bf16  = silu(acc(W)) * acc(W2)    */
  SX_EPI_SWIGLU_IL = 4,   /* W = [gate; up] interleaved in 64-row blocks (rows 128j..128j+63 =
                             gate features 64j.., rows 128j+64.. = up of the same features);
                             out bf16 [M, N/2] = silu(gate) * up   (N % 128 == 0)      */
  SX_EPI_RS_BF16 = 5,     /* internal: the reduce-scatter epilogue of sx_gemm_bf16_rs        */
  SX_EPI_QKV_ROPE = 6     /* internal: the RoPE + KV-scatter epilogue of sx_gemm_qkv_rope    */
};
/* 0 = auto (default: CTA-pair cta_group::2 tiles for M >= 256 tokens), 1 = single-CTA only, 2 = pair when legal */
SX_API int sx_gemm_set_pair_mode(int mode);
/* 1 (default) = M <= 4 tokens run the weight-streaming matrix-vector kernel (same
 * epilogues except SWIGLU_BF16 / RS_BF16); 0 = always the tcgen05 tile kernel (A/B) */
SX_API int sx_gemm_set_gemv(int enabled);
SX_API int sx_gemm_plan(int M, int N, int K, int dual, int splits_req, int* bn_out, int* splits_out,
                 long long* ws_floats_out);
SX_API int sx_gemm_bf16(const void* W, const void* W2, const void* X, void* out, float* ws, long long ws_floats,
                 int M, int N, int K, long long ldo, int epi, int splits_req, cudaStream_t stream);
/* Tensor-parallel row-parallel projection fused with the reduce-scatter half of
 * its all-reduce: this rank's partial Y = X W^T (bf16) is written by the GEMM
 * epilogue straight into the owners' inboxes over NVLink peer memory:
 * feature f -> rank f / (N/world), at peer_inbox[owner] + ((rank * M + t) * (N/world)
 * + f % (N/world)). peer_inbox: DEVICE array of `world` pointers (symmetric
 * memory, [world][M][N/world] bf16 each). Then, after a cross-rank barrier,
 * sx_tp_reduce_bcast on every rank sums its slice in rank order and writes it into
 * every rank's y [M, N] (the all-gather half). Deterministic; identical on all ranks. */
SX_API int sx_gemm_bf16_rs(const void* W, const void* X, void* const* peer_inbox, int rank, int world, float* ws,
                           long long ws_floats, int M, int N, int K, int splits_req, cudaStream_t stream);
/* QKV projection with RoPE and the KV-cache scatter fused into the epilogue
 * (replaces sx_gemm_bf16 + sx_rope_kv): W [(H + 2 KVH) * 128, K] (q heads, k
 * heads, v heads); each 128-row tile is one head, rotated (rotate-half, position
 * pos_base + pos[t], tables [max_pos, 64]) from the fp32 accumulator and stored
 * to q [M, H, 128] or to cache slot slot_base + slot[t] of K / V [KVH][slots][128]. */
SX_API int sx_gemm_qkv_rope(const void* W, const void* X, float* ws, long long ws_floats, int M, int H, int KVH, int K,
                            const int* pos, int pos_base, const int* slot, int slot_base, const float* cos_t,
                            const float* sin_t, void* q, void* kcache, void* vcache, long long slots, int splits_req,
                            cudaStream_t stream);
SX_API int sx_tp_reduce_bcast(const void* inbox, int rank, int world, int M, int N, void* const* peer_y, int y_bf16,
                              cudaStream_t stream);

/* ------------------------------------- KT1-KT3: draft-tree build (stage 1)
 * build_sssp, pkg/src/speckit/tree.py:240-327, as a device-resident state
 * machine in one caller-allocated workspace of sx_tree_workspace_bytes(K,B,V,D)
 * bytes (K = budget, B = batch_size, V = vocab, D = max_depth; BuilderParams
 * tree.py:36-55). Per draft call the caller evaluates the draft on the current
 * batch (its tokens / ancestor KV slots are in the workspace, see
 * sx_tree_offsets) and hands the rows to sx_tree_round, which scores them
 * (tree.py:299-306; warp per _scored_dist tree.py:222-227), keeps the K best by
 * (nll, depth, path-lex) (tree.py:308-318) and selects the next batch
 * (tree.py:282-295). `host_ctl` (pinned, >= 64 bytes) receives the control
 * block (batch size == 0 ends the build). sx_tree_finalize lays the result out
 * in node-id order (ids in key order, tree.py:320-327).
 */
/* SX_ROWS_ARGMAX_PACKED: one int64 key per row (sx_rows_argmax_packed, max-reduced
 * over vocab shards): the row's argmax for t = 0 walks (KV1) */
enum { SX_ROWS_LOGITS_F32 = 0, SX_ROWS_PROBS_F64 = 1, SX_ROWS_ARGMAX_PACKED = 2 };
enum { SX_SCORE_RAW = 0, SX_SCORE_ARGMAX = 1, SX_SCORE_WARP = 2 };
SX_API long long sx_tree_workspace_bytes(int K, int B, int V, int D);
/* byte offsets into the workspace, in this order: ctl, b_node, b_nll, b_depth, b_lex,
 * b_slot, b_token, b_anc, b_anc_len, f_anc, f_anc_len, f_depth, f_token, w_rows,
 * b_pos, b_dense, total, r_aux; returns the number of offsets available */
SX_API int sx_tree_offsets(int K, int B, int V, int D, long long* out, int n);
SX_API int sx_tree_begin(void* ws, int K, int B, int V, int D, int root_slot, int pad_slot,
                         cudaStream_t stream);
SX_API int sx_tree_round(void* ws, int K, int B, int V, int D, const void* rows, int row_kind, long long ld,
                         int score_mode, double temperature, double top_p, int* host_ctl, cudaStream_t stream);
SX_API int sx_tree_finalize(void* ws, int K, int B, int V, int D, int root_token, int* out_parent, int* out_token,
                            double* out_edge, int* out_depth, int* out_slot, cudaStream_t stream);
/* Raw scoring of fp32 logits rows: 0 (default) = the chunked path (max / sum /
 * score kernels over (row, chunk) units, one HBM read per prefiltered row), 1 =
 * the two-kernel tree_row_stats + tree_score path (A/B; identical results). */
SX_API int sx_tree_set_impl(int unfused);
/* Survivor buffer (candidates of one round that beat the threshold): capacity
 * min(B*V, max(V + K, 2^24)) entries (sx_tree_survivor_cap). A round whose
 * survivors overflow it leaves the tree untouched and reports ctl->err (int 8
 * of host_ctl); the caller then clears the flag (sx_tree_clear_overflow) and
 * re-runs the SAME rows in slices [r0, r1) of at most cap / V rows with
 * sx_tree_round_rows: final = 0 merges a slice's survivors (keeping the K best,
 * remapping the batch), final = 1 on the last slice also picks the next batch --
 * the same tree as one unbounded round. sx_tree_round == rows [0, batch_n),
 * final = 1. sx_tree_set_survivor_cap overrides the capacity of workspaces
 * laid out afterwards (0 = default; tests). */
SX_API long long sx_tree_survivor_cap(int K, int B, int V, int D);
SX_API int sx_tree_set_survivor_cap(long long cap);
SX_API int sx_tree_clear_overflow(void* ws, int K, int B, int V, int D, cudaStream_t stream);
SX_API int sx_tree_round_rows(void* ws, int K, int B, int V, int D, const void* rows, int row_kind, long long ld,
                              int score_mode, double temperature, double top_p, int r0, int r1, int final,
                              int* host_ctl, cudaStream_t stream);

/* ------------------------------------------------ exact table models on GPU
 * MarkovModel / TabularModel (pkg/src/speckit/models.py:77-151) rows for tree
 * nodes: table fp64 [V**order, V]; ctx0 = anchor's last `order` tokens
 * left-padded with 0 (device int[order]); node_ids = positions in the tree
 * workspace's current node list or -1 for the anchor (or from_batch=1: the
 * current batch). out fp64 [n, ld].
 */
SX_API int sx_markov_rows(const double* table, int V, int order, const int* ctx0, void* ws, int K, int B, int D,
                          const int* node_ids, int n_nodes, int from_batch, double* out, long long ld,
                          cudaStream_t stream);

/* ---------------------------------------- KV1/KV2: verification (stage 4)
 * The acceptance walk of generate_specexec (pkg/src/speckit/engine.py:118-128):
 * rows = target rows of the flattened tree (row 0 = anchor, row i+1 = node i;
 * fp32 logits or fp64 probabilities); parent/token = the tree in node-id
 * order. Per step: token = sample(apply_warp(row[cursor]), uniforms[step])
 * (sampling.py:66-113; t = 0 -> argmax, lowest id); move to the child with that
 * token (tree.py:132-136); stop on a miss or after max_steps.
 * out (device int[3 + 2*max_steps]): [emitted, fell_off, cursor, tokens..., path rows...].
 * scratch: sx_row_scratch_bytes(V) bytes.
 */
SX_API long long sx_row_scratch_bytes(int V);
SX_API int sx_verify_walk(const void* rows, int row_kind, long long ld, int V, const int* parent, const int* token,
                          int n_nodes, int start_cursor, const double* uniforms, int max_steps, double temperature,
                          double top_p, int* out, void* scratch, cudaStream_t stream);
/* apply_warp (sampling.py:66-98) of n rows (row_ids may be NULL) into fp64 out [n, ldo];
 * scratch: sx_warp_scratch_bytes(n, V). */
SX_API long long sx_warp_scratch_bytes(int n, int V);
SX_API int sx_warp_rows(const void* rows, int row_kind, long long ld, int V, const int* row_ids, int n,
                        double temperature, double top_p, double* out, long long ldo, void* scratch,
                        cudaStream_t stream);
/* canonical float64 probabilities of fp32 logits rows (ProbCache row materialisation) */
SX_API int sx_softmax_rows(const float* rows, long long ld, int V, const int* row_ids, int n, double* out,
                           long long ldo, cudaStream_t stream);
SX_API int sx_argmax_rows(const void* rows, int row_kind, long long ld, int V, int n, int* out, cudaStream_t stream);
/* KV1 (vocab-parallel LM head, t = 0): out[r] = max over v in the slice of
 * orderable(logits[r][v]) << 31 | (0x7fffffff - (v0 + v)); an int64 MAX all-reduce
 * of these keys over the shards gives the global argmax (lowest id on ties).
 * Replaces the all-gather of the logit slices (engine.py:124 at t = 0). */
SX_API int sx_rows_argmax_packed(const float* logits, long long ld, int n, int Vl, int v0, long long* out,
                                 cudaStream_t stream);
/* sample (sampling.py:101-113) from n warped fp64 rows with uniforms u[n] */
SX_API int sx_sample_rows(const double* w, long long ld, int V, const double* u, int n, int* out,
                          cudaStream_t stream);

/* ------------------------------------------ KB1/KB2: beam search (8(f) row 4)
 * One step of build_beam (pkg/src/speckit/tree.py:330-380): q = the beams'
 * scored rows (fp64 [nb, ldq]), beam_nll / beam_rank (lex rank of each beam's
 * path) per beam; keeps the beam_size best candidates by (nll, path).
 * scratch: sx_beam_scratch_bytes(nb, V); c_* per-row candidate buffers
 * [nb * beam_size] (c_cnt [nb]); out_* [beam_size], out_n: kept count.
 * nb * beam_size <= 8192. */
SX_API long long sx_beam_scratch_bytes(int nb, int V);
SX_API int sx_beam_step(const double* q, long long ldq, int V, int nb, const double* beam_nll, const int* beam_rank,
                        int beam_size, void* scratch, double* c_nll, double* c_edge, int* c_tok, int* c_cnt,
                        int* out_n, double* out_nll, double* out_edge, int* out_beam, int* out_tok,
                        cudaStream_t stream);

/* ------------------------------------ KI1/KI2: SpecInfer baseline (8(f) row 1)
 * build_stochastic's draws (pkg/src/speckit/tree.py:383-425): token[i] =
 * sample(w[row_ids[i]], u[i]) and out_logq[i] = log w[row][token] (may be NULL).
 * verify_specinfer (pkg/src/speckit/specinfer.py:53-96) as one CTA: tree rows
 * trows (row 0 = anchor, row n+1 = node n); per row r the children are node ids
 * [child_start[r], +child_count[r]) drawn from q[q_row[r]] (fp64 [*, ldq]);
 * token / mult per node; uniforms = the "specinfer-accept" stream (n_u of them,
 * an upper bound). out (device int[4 + max_path]): [path_len, bonus_token,
 * uniforms_used, error (0 ok, 1 residual invalid, 2 missing q, 3 uniforms
 * exhausted), path node ids...]. scratch: sx_row_scratch_bytes(V).
 */
SX_API int sx_sample_rows_idx(const double* w, long long ld, int V, const int* row_ids, const double* u, int n,
                              int* out_tok, double* out_logq, cudaStream_t stream);
SX_API int sx_specinfer_verify(const void* trows, int row_kind, long long ld, int V, const double* q, long long ldq,
                               const int* q_row, const int* child_start, const int* child_count, const int* token,
                               const int* mult, int max_path, const double* uniforms, int n_u, double temperature,
                               double top_p, int* out, void* scratch, cudaStream_t stream);

/* ------------------------------------------- KE / KA / KV3: model forward
 * Llama-shaped forward used for the draft rounds (stage 1) and the single
 * target pass over the flattened tree (stage 2); together they implement
 * LanguageModel.next_distributions (pkg/src/speckit/models.py:47-52) for the
 * B200 models. KV cache per layer: K and V [KVH][slots][128] bf16.
 *   sx_embed      x[t] = float(E[tokens[t]])                    (fp32 residual)
 *   sx_rmsnorm    y = bf16(x * rsqrt(mean(x^2) + eps) * w)
 *   sx_add_rmsnorm x += y (y fp32, or bf16 when y_bf16), then out = bf16(x * rsqrt(mean(x^2) + eps) * w);
 *                 w NULL: the residual add only
 *   sx_rope_kv    rotate-half RoPE of q/k at pos_base + pos[t]; q -> [n,H,128];
 *                 k,v -> cache slot slot_base + slot[t] (pos/slot NULL: t)
 *   sx_tree_attention  query t attends KV slots [0, dense_len[t]) (NULL: dense_const)
 *                 plus the anc_len[t] slots anc_base + anc[t*A ...] (root, ancestors, itself) -- the
 *                 flattened ancestor mask of tree.py:208-219 without a dense mask
 *   sx_kv_compact move KV rows src[i] -> dst[i] (n <= 448) in every layer / head (accepted
 *                 path -> committed region after the walk)
 */
SX_API int sx_embed(const void* E, const int* tokens, int n, int d, float* x, cudaStream_t stream);
SX_API int sx_rmsnorm(const float* x, const void* w, int n, int d, float eps, void* y, cudaStream_t stream);
SX_API int sx_add_rmsnorm(float* x, const void* y, int y_bf16, const void* w, int n, int d, float eps, void* out,
                          cudaStream_t stream);
SX_API int sx_rope_kv(const void* qkv, const int* pos, int pos_base, const int* slot, int slot_base, int n, int H,
                      int KVH, const float* cos_t, const float* sin_t, void* q, void* kcache, void* vcache,
                      long long slots, cudaStream_t stream);
SX_API int sx_tree_attention(const void* q, const void* kcache, const void* vcache, long long slots,
                             const int* dense_len, int dense_const, const int* anc, int anc_base, const int* anc_len,
                             int A, void* out, int N, int H, int KVH, cudaStream_t stream);
/* Same, with a workspace for the key-split path of the tcgen05 kernel (small
 * grids: one-token steps, small batches): ws_bytes >= sx_tree_attention_ws_bytes
 * (0 = the shape needs none; NULL / too small = no split). The workspace must be
 * zero-filled before its first use (it holds arrival counters the kernel resets);
 * one workspace per stream. */
SX_API long long sx_tree_attention_ws_bytes(int N, int H, int KVH);
SX_API int sx_tree_attention_ws(const void* q, const void* kcache, const void* vcache, long long slots,
                                const int* dense_len, int dense_const, const int* anc, int anc_base,
                                const int* anc_len, int A, void* out, int N, int H, int KVH, void* ws,
                                long long ws_bytes, cudaStream_t stream);
/* Attention kernel selection: 0 = by shape (default: the tcgen05/TMEM kernel
 * unless the batch is a small MHA batch or a one-token step), 1 = the 64-row
 * mma.sync flash loop only, 2 = the tcgen05 kernel only (A/B measurement). */
SX_API int sx_attention_set_impl(int impl);
/* ------------------------------------------------ KS: weight streaming (stage 3)
 * Async copy of `bytes` between pinned host memory and device memory on
 * `stream` (to_device = 1: H2D), after waiting on `wait_event` (may be NULL) and
 * recording `done_event` (may be NULL) -- the double-buffer handshake of the
 * offloaded target (modelled by costsim.forward_time, pkg/src/speckit/costsim.py:59-65).
 */
SX_API int sx_stream_copy(void* dst, const void* src, long long bytes, int to_device, cudaStream_t stream,
                          cudaEvent_t wait_event, cudaEvent_t done_event);
SX_API int sx_kv_compact(void* kcache, void* vcache, int layers, long long layer_stride, long long slots, int KVH,
                         const int* src, const int* dst, int n, cudaStream_t stream);

/* ------------------------------------------------ fp32 target mode (csrc/fp32_path.cu)
 * The same forward with fp32 weights, activations, KV cache and CUDA-core FFMA
 * accumulation (north_star: target logits within 1e-4 of the fp32 reference).
 * Semantics as the bf16 entry points above; all pointers fp32.
 *   sx_gemm_f32        out[t, f] (op)= sum_k x[t, k] w[f, k]; epi SX_EPI_F32 / SX_EPI_ADD_F32 /
 *                      SX_EPI_SWIGLU_IL (out [M, N/2]); K a multiple of 4, 16-byte aligned operands
 *   sx_tree_attention_f32  key set as sx_tree_attention (H / KVH <= 32)
 *   sx_add_rmsnorm_f32 x += y (y NULL: none), out = x * rsqrt(mean(x^2) + eps) * w (w NULL: add only)
 *   sx_kv_compact_f32  as sx_kv_compact on an fp32 cache (n <= 224)
 */
SX_API int sx_gemm_f32(const float* w, const float* x, float* out, int M, int N, int K, long long ldo, int epi,
                       cudaStream_t stream);
SX_API int sx_tree_attention_f32(const float* q, const float* kcache, const float* vcache, long long slots,
                                 const int* dense_len, int dense_const, const int* anc, int anc_base,
                                 const int* anc_len, int A, float* out, int N, int H, int KVH, cudaStream_t stream);
SX_API int sx_embed_f32(const float* E, const int* tokens, int n, int d, float* x, cudaStream_t stream);
SX_API int sx_add_rmsnorm_f32(float* x, const float* y, const float* w, int n, int d, float eps, float* out,
                              cudaStream_t stream);
SX_API int sx_rope_kv_f32(const float* qkv, const int* pos, int pos_base, const int* slot, int slot_base, int n,
                          int H, int KVH, const float* cos_t, const float* sin_t, float* q, float* kcache,
                          float* vcache, long long slots, cudaStream_t stream);
SX_API int sx_kv_compact_f32(void* kcache, void* vcache, int layers, long long layer_stride, long long slots,
                             int KVH, const int* src, const int* dst, int n, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SPECEXEC_B200_H_ */
