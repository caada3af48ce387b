// Device workspace layout of the stage-1 draft-tree builder (build_sssp,
// pkg/src/speckit/tree.py:240-327). One flat byte buffer (allocated by the
// caller) holds every array; offsets are computed identically on host and
// device from (K, B, V, D).
#pragma once
#include <stdint.h>

namespace sx {

struct TreeCtl {
  int cur;         // which materialized buffer (0/1) is current
  int count;       // materialized nodes (<= K), sorted by key in buffer `cur`
  int has_thr;     // threshold valid (count == K)
  int rounds;      // draft calls so far (tree.rounds)
  int slot_next;   // next free draft-KV slot
  int batch_n;     // nodes in the current batch
  int n_surv;      // candidates appended by the scorer this round
  int root_slot;   // draft-KV slot of the root (anchor's last token)
  int err;         // 1 = survivor buffer overflow
  int pad_slot;    // KV slot that padded batch rows (b >= batch_n) write to
  double thr_nll;
  unsigned long long thr_lo;
};

struct TreeLayout {
  int K, B, V, D, kpad;
  long long cap;  // survivor capacity
  // byte offsets
  long long ctl;
  long long m_nll[2], m_lo[2], m_edge[2], m_parent[2], m_lex[2], m_slot[2];
  long long b_node, b_nll, b_depth, b_lex, b_slot, b_token, b_anc, b_anc_len, b_pos, b_dense;
  long long s_nll, s_lo, s_edge, s_row;
  long long remap;
  long long r_max, r_sum;
  long long w_rows;     // fp64 [B, V] warped rows (t > 0 scoring)
  long long w_keys, w_idx, w_keys2, w_idx2;  // [wsc, V] sort scratch, one row per CTA of the warp kernel
  int wsc;              // CTAs (scratch rows) of tree_warp_rows_kernel = min(B, kWarpScratchRows)
  long long f_anc, f_anc_len, f_depth, f_token;  // final target-row tables [(K+1)]
  long long r_lsa;      // float [B]: fp32 log-sum-exp estimate (threshold prefilter), -inf: row skipped
  // chunked logits-row path (tree_rows_{max,sum,score}_kernel)
  long long r_pm, r_ps;  // float [B][kRowChunksMax]: per-chunk max / fp32 sum of exp(z - max)
  long long r_cnt;       // int [2][B]: chunk arrival counters (max pass, sum pass); reset by the last arriver
  long long r_list;      // int [B]: rows that need the exact passes (not prefiltered away)
  long long r_ready;     // int [B]: fused exact pass: row sum published for round stamp r_aux[1] + 1
  long long r_aux;       // int [64]: [0] = rows in r_list, [1] = round stamp (never reset), [16..48) trace
  long long total;
};

constexpr int kWarpScratchRows = 148;  // one warp-row CTA per SM (its shared-memory radix histograms fill the SM)
constexpr int kRowChunkA = 4096;  // elements per work unit of the max pass
constexpr int kRowChunkB = 1024;  // elements per work unit of the exp / score passes
constexpr int kRowChunksMax = 64;  // V <= 262144 -> <= 64 max-pass chunks per row

__host__ __device__ inline long long tl_align(long long x) { return (x + 255) & ~255LL; }

// Survivor capacity (candidates of one round that beat the threshold): B x V
// bounds it, but only a first round without a threshold (<= V of the root) or
// very flat rows come near it; 2^24 entries (448 MB) cover every measured round.
// A round that still overflows is re-run in row slices (sx_tree_round_rows).
constexpr long long kSurvivorCapMin = 1LL << 24;

inline long long default_survivor_cap(int K, int B, int V) {
  const long long full = (long long)B * V;
  long long cap = (long long)V + K;
  if (cap < kSurvivorCapMin) cap = kSurvivorCapMin;
  return cap < full ? cap : full;
}

inline TreeLayout tree_layout(int K, int B, int V, int D, long long cap) {
  TreeLayout L{};
  L.K = K;
  L.B = B;
  L.V = V;
  L.D = D;
  int kp = 1;
  while (kp < K) kp <<= 1;
  L.kpad = kp;
  L.cap = cap;
  long long o = 0;
  auto take = [&](long long bytes) {
    long long r = o;
    o = tl_align(o + bytes);
    return r;
  };
  L.ctl = take(sizeof(TreeCtl));
  for (int i = 0; i < 2; ++i) {
    L.m_nll[i] = take(8LL * K);
    L.m_lo[i] = take(8LL * K);
    L.m_edge[i] = take(8LL * K);
    L.m_parent[i] = take(4LL * K);
    L.m_lex[i] = take(4LL * K);
    L.m_slot[i] = take(4LL * K);
  }
  L.b_node = take(4LL * B);
  L.b_nll = take(8LL * B);
  L.b_depth = take(4LL * B);
  L.b_lex = take(4LL * B);
  L.b_slot = take(4LL * B);
  L.b_token = take(4LL * B);
  L.b_anc = take(4LL * B * (D + 1));
  L.b_anc_len = take(4LL * B);
  L.b_pos = take(4LL * B);
  L.b_dense = take(4LL * B);
  L.s_nll = take(8LL * L.cap);
  L.s_lo = take(8LL * L.cap);
  L.s_edge = take(8LL * L.cap);
  L.s_row = take(4LL * L.cap);
  L.remap = take(4LL * K);
  L.r_max = take(4LL * B);
  L.r_sum = take(8LL * B);
  L.w_rows = take(8LL * B * V);
  L.wsc = B < kWarpScratchRows ? B : kWarpScratchRows;
  L.w_keys = take(8LL * L.wsc * V);
  L.w_idx = take(4LL * L.wsc * V);
  L.w_keys2 = take(8LL * L.wsc * V);
  L.w_idx2 = take(4LL * L.wsc * V);
  L.f_anc = take(4LL * (K + 1) * (D + 1));
  L.f_anc_len = take(4LL * (K + 1));
  L.f_depth = take(4LL * (K + 1));
  L.f_token = take(4LL * (K + 1));
  L.r_lsa = take(4LL * B);
  L.r_pm = take(4LL * B * kRowChunksMax);
  L.r_ps = take(4LL * B * kRowChunksMax);
  L.r_cnt = take(8LL * B);
  L.r_list = take(4LL * B);
  L.r_ready = take(4LL * B);
  L.r_aux = take(4LL * 64);
  L.total = o;
  return L;
}

}  // namespace sx
