// KA: tree-masked attention for the draft rounds and the target pass over the
// flattened tree.
//
// The reference's verification mask is `flatten`'s dense ancestor matrix
// (pkg/src/speckit/tree.py:208-219): position i sees the anchor prefix, the
// root, its ancestors and itself. Here that mask is never materialised. Each
// query token carries
//   dense_len  : it attends to KV slots [0, dense_len) (the committed prefix;
//                for causal prefill chunks dense_len = own slot + 1), and
//   anc[0..n)  : an explicit list of extra KV slots (root + tree ancestors +
//                itself; <= max_depth + 1 entries).
// Two kernels share that key-space scheme: the tcgen05 kernel (128 rows per
// CTA, S and O accumulated in TMEM; below) for tree passes and prefill, and a
// 64-row mma.sync flash loop for small MHA batches and one-token steps
// (selection in sx_tree_attention). The mma.sync loop: bf16 m16n8k16, fp32
// online softmax, cp.async double-buffered K/V tiles, XOR-swizzled shared
// memory; one key space: the committed prefix [0, maxlen)
// followed by the ancestor keys gathered by slot -- the concatenated ancestor
// lists of the CTA's tokens (<= D+1 keys each), each row masked to its own
// segment -- so the ancestors fill the last partial committed tile. GQA:
// one CTA serves one KV head and 64 query rows = (64 / G) tokens x G heads.
#include <cstdlib>

#include "capi_util.h"
#include "common.cuh"
#include "specexec_b200.h"

namespace sx {

constexpr int kAttRows = 64;
constexpr int kAttWarps = 4;
constexpr int kKeyTile = 64;
constexpr int kHd = 128;

struct AttnArgs {
  const __nv_bfloat16* q;
  const __nv_bfloat16* kc;
  const __nv_bfloat16* vc;
  long long slots;
  const int* dense_len;
  int dense_const;
  int anc_base;
  const int* anc;
  const int* anc_len;
  int A;
  __nv_bfloat16* out;
  int N, H, KVH, G, QB;
  float scale_log2;
  float rescale_thresh;  // tcgen05 kernel: move the running max only when it grows by more (log2 units)
  int splits;            // tcgen05 kernel: key splits (gridDim.z); > 1 writes partials to `part`
  float* part;           // [q tiles][KVH][splits][128 rows][kPartStride] fp32 (O, m, l)
  int* counters;         // [q tiles][KVH] split arrival counts (zero between launches)
};

SX_DEV uint32_t swz(int row, int col) {  // byte offset inside a [rows][128] bf16 tile
  const int chunk = (col >> 3) ^ (row & 7);
  return row * 256 + chunk * 16 + (col & 7) * 2;
}

SX_DEV void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
SX_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
SX_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

SX_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
SX_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
SX_DEV void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
SX_DEV uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

constexpr int kMaxAncKeys = 64 * 32;  // QB tokens x A ancestors (A <= 32)

struct AttnSmem {
  uint8_t qs[kAttRows * 256];
  uint8_t ks[2][kKeyTile * 256];
  uint8_t vs[2][kKeyTile * 256];
  int dlen[kAttRows];
  int seg[kAttRows + 1];  // per token of the CTA: start of its ancestor segment
  int aslot[kMaxAncKeys];
  int maxlen;
};

__global__ void __launch_bounds__(kAttWarps * 32) tree_attention_kernel(const AttnArgs a) {
  griddep_launch_dependents();
  extern __shared__ __align__(128) uint8_t smem_raw[];
  AttnSmem& sm = *reinterpret_cast<AttnSmem*>(smem_raw);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kvh = blockIdx.y;
  const int t0 = blockIdx.x * a.QB;
  const __nv_bfloat16* kbase = a.kc + (long long)kvh * a.slots * kHd;
  const __nv_bfloat16* vbase = a.vc + (long long)kvh * a.slots * kHd;

  if (tid == 0) sm.maxlen = 0;
  __syncthreads();
  if (tid < kAttRows) {
    const int t = t0 + tid / a.G;
    const int dl = t < a.N ? (a.dense_len ? a.dense_len[t] : a.dense_const) : 0;
    sm.dlen[tid] = dl;
    atomicMax(&sm.maxlen, dl);
  }
  if (tid < a.QB) {  // ancestor counts, loaded in parallel
    const int t = t0 + tid;
    sm.seg[tid + 1] = (t < a.N && a.anc_len) ? a.anc_len[t] : 0;
  }
  __syncthreads();
  if (tid == 0) {  // ancestor segments of the CTA's tokens (prefix sum over smem, <= 64 tokens)
    sm.seg[0] = 0;
    for (int i = 1; i <= a.QB; ++i) sm.seg[i] += sm.seg[i - 1];
  }
  __syncthreads();
  const int n_anc = sm.seg[a.QB];
  for (int i = tid; i < a.QB * a.A; i += blockDim.x) {
    const int tl = i / a.A, j = i % a.A, t = t0 + tl;
    if (t < a.N && j < sm.seg[tl + 1] - sm.seg[tl])
      sm.aslot[sm.seg[tl] + j] = a.anc_base + a.anc[(long long)t * a.A + j];
  }
  // Q tile: rows r = token-major, head-minor
  const uint32_t qs = smem_u32(sm.qs);
  for (int i = tid; i < kAttRows * 16; i += blockDim.x) {
    const int r = i >> 4, c = i & 15;
    const int t = t0 + r / a.G, h = kvh * a.G + r % a.G;
    const __nv_bfloat16* src = a.q + ((long long)(t < a.N ? t : 0) * a.H + h) * kHd + c * 8;
    cp_async16(qs + swz(r, c * 8), src, t < a.N ? 16 : 0);
  }
  cp_async_commit();
  __syncthreads();
  const int maxlen = sm.maxlen;
  // one key space: committed slots [0, maxlen) followed by the ancestor keys
  // [maxlen, maxlen + n_anc) -- the ancestors fill the last partial dense tile
  const int ntiles = (maxlen + n_anc + kKeyTile - 1) / kKeyTile;

  auto load_kv = [&](int tile, int buf) {
    const uint32_t ks = smem_u32(sm.ks[buf]), vs = smem_u32(sm.vs[buf]);
    for (int i = tid; i < kKeyTile * 16; i += blockDim.x) {
      const int r = i >> 4, c = i & 15;
      const int key = tile * kKeyTile + r;
      long long slot;
      bool ok;
      if (key < maxlen) {
        ok = true;
        slot = key;
      } else {
        const int k = key - maxlen;
        ok = k < n_anc;
        slot = ok ? sm.aslot[k] : 0;
      }
      const long long off = slot * kHd + c * 8;
      cp_async16(ks + swz(r, c * 8), kbase + off, ok ? 16 : 0);
      cp_async16(vs + swz(r, c * 8), vbase + off, ok ? 16 : 0);
    }
    cp_async_commit();
  };
  if (ntiles > 0) load_kv(0, 0);

  // per-thread state: rows ra = warp*16 + lane/4, rb = ra + 8
  const int ra = warp * 16 + (lane >> 2), rb = ra + 8;
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_a = -1e30f, m_b = -1e30f, l_a = 0.f, l_b = 0.f;
  uint32_t qf[8][4];

  cp_async_wait<1>();  // Q landed (K/V tile 0 may still be in flight)
  if (ntiles == 0) cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    const int r = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
    const int c = ks * 16 + (lane >> 4) * 8;
    ldsm_x4(qs + swz(r, c), qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3]);
  }
  const int dl_a = sm.dlen[ra], dl_b = sm.dlen[rb];
  const int sa_lo = sm.seg[ra / a.G], sa_hi = sm.seg[ra / a.G + 1];
  const int sb_lo = sm.seg[rb / a.G], sb_hi = sm.seg[rb / a.G + 1];

  for (int kt = 0; kt < ntiles; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < ntiles) {
      load_kv(kt + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint32_t ksm = smem_u32(sm.ks[buf]), vsm = smem_u32(sm.vs[buf]);
    float s[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 8; ks += 2) {
        uint32_t b0, b1, b2, b3;
        const int r = nt * 8 + (lane & 7);
        const int c = ks * 16 + (lane >> 3) * 8;
        ldsm_x4(ksm + swz(r, c), b0, b1, b2, b3);
        mma_bf16(s[nt], qf[ks], b0, b1);
        mma_bf16(s[nt], qf[ks + 1], b2, b3);
      }
    }
    // mask: committed key < dense_len of the row, or an ancestor key in the row's own segment
    const int kb = kt * kKeyTile;
    const int alo_a = maxlen + sa_lo, ahi_a = maxlen + sa_hi, alo_b = maxlen + sb_lo, ahi_b = maxlen + sb_hi;
    float mx_a = -INFINITY, mx_b = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int key = kb + nt * 8 + (lane & 3) * 2;
      const bool a0 = key < dl_a || (key >= alo_a && key < ahi_a);
      const bool a1 = key + 1 < dl_a || (key + 1 >= alo_a && key + 1 < ahi_a);
      const bool b0 = key < dl_b || (key >= alo_b && key < ahi_b);
      const bool b1 = key + 1 < dl_b || (key + 1 >= alo_b && key + 1 < ahi_b);
      s[nt][0] = a0 ? s[nt][0] * a.scale_log2 : -INFINITY;
      s[nt][1] = a1 ? s[nt][1] * a.scale_log2 : -INFINITY;
      s[nt][2] = b0 ? s[nt][2] * a.scale_log2 : -INFINITY;
      s[nt][3] = b1 ? s[nt][3] * a.scale_log2 : -INFINITY;
      mx_a = fmaxf(mx_a, fmaxf(s[nt][0], s[nt][1]));
      mx_b = fmaxf(mx_b, fmaxf(s[nt][2], s[nt][3]));
    }
    mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffff, mx_a, 1));
    mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffff, mx_a, 2));
    mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffff, mx_b, 1));
    mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffff, mx_b, 2));
    const float mn_a = fmaxf(m_a, mx_a), mn_b = fmaxf(m_b, mx_b);
    const float ca = exp2f(m_a - mn_a), cb = exp2f(m_b - mn_b);
    m_a = mn_a;
    m_b = mn_b;
    float sa = 0.f, sb = 0.f;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      s[nt][0] = exp2f(s[nt][0] - mn_a);
      s[nt][1] = exp2f(s[nt][1] - mn_a);
      s[nt][2] = exp2f(s[nt][2] - mn_b);
      s[nt][3] = exp2f(s[nt][3] - mn_b);
      sa += s[nt][0] + s[nt][1];
      sb += s[nt][2] + s[nt][3];
    }
    sa += __shfl_xor_sync(0xffffffff, sa, 1);
    sa += __shfl_xor_sync(0xffffffff, sa, 2);
    sb += __shfl_xor_sync(0xffffffff, sb, 1);
    sb += __shfl_xor_sync(0xffffffff, sb, 2);
    l_a = l_a * ca + sa;
    l_b = l_b * cb + sb;
#pragma unroll
    for (int nd = 0; nd < 16; ++nd) {
      o[nd][0] *= ca;
      o[nd][1] *= ca;
      o[nd][2] *= cb;
      o[nd][3] *= cb;
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t pa[4];
      pa[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int nd = 0; nd < 16; nd += 2) {
        uint32_t b0, b1, b2, b3;
        const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = nd * 8 + (lane >> 4) * 8;
        ldsm_x4_t(vsm + swz(r, c), b0, b1, b2, b3);
        mma_bf16(o[nd], pa, b0, b1);
        mma_bf16(o[nd + 1], pa, b2, b3);
      }
    }
    __syncthreads();
  }

  // normalise and store: rows ra / rb, dims nd*8 + (lane&3)*2 (+1)
  const float inv_a = l_a > 0.f ? 1.f / l_a : 0.f, inv_b = l_b > 0.f ? 1.f / l_b : 0.f;
  const int ta = t0 + ra / a.G, tb = t0 + rb / a.G;
  __nv_bfloat16* da = a.out + ((long long)ta * a.H + kvh * a.G + ra % a.G) * kHd;
  __nv_bfloat16* db = a.out + ((long long)tb * a.H + kvh * a.G + rb % a.G) * kHd;
#pragma unroll
  for (int nd = 0; nd < 16; ++nd) {
    const int c = nd * 8 + (lane & 3) * 2;
    if (ta < a.N) *reinterpret_cast<uint32_t*>(da + c) = pack_bf16(o[nd][0] * inv_a, o[nd][1] * inv_a);
    if (tb < a.N) *reinterpret_cast<uint32_t*>(db + c) = pack_bf16(o[nd][2] * inv_b, o[nd][3] * inv_b);
  }
}


// ---------------------------------------------------------------------------
// tcgen05 variant: 128 query rows per CTA ((128 / G) tokens x G heads of one KV
// head), the whole tile in one MMA per 16-wide k step, accumulators in TMEM.
//
//   S  (TMEM cols [0, 64))    = Q K^T            M=128 N=64  K=128 (8 MMAs)
//   O  (TMEM cols [64, 192)) += P V              M=128 N=128 K=64  (4 MMAs)
//
// Two threads own query row r = TMEM lane r (warps w and w + 4 share a lane
// quadrant), one per half of the 64 key columns / 128 output dims: each reads
// its half of the S row (tcgen05.ld), masks and exponentiates it (the row max
// is exchanged through shared memory), and writes its half of the P row (bf16)
// into the K buffer of the same tile (K is dead once S has been computed). When the row
// max grows, O is rescaled in TMEM (a warp-collective ld/scale/st round trip,
// skipped by warps whose rows kept their max). Q, K, V and P live in smem
// in the canonical 128B-swizzled layouts: Q / K / P K-major (rows of 64 bf16),
// V MN-major (a key's 128 dims are two 128-byte rows, LBO = 8 KB between them),
// so V is read straight from the cache layout without a transpose. K/V tiles
// (committed slots, then the ancestor slots gathered by id) are double-buffered
// with cp.async; tile kt+1 is fetched while tile kt is in softmax and P V.
constexpr int kTcRows = 128;
constexpr int kTcThreads = 256;  // 2 threads per query row (column halves)
constexpr uint32_t kTcTmemCols = 256;
// Move the running max (and rescale O in TMEM) whenever it grows. A lazy
// threshold of 8 (FA4-style, P <= 256) was measured: no speed-up on the
// SpecExec shapes (<= 8 % on 1k-key contexts) but 1.6-2x the max abs error of
// the exact-max path vs an fp32 reference (tools/attn_err.py), so exact it is.
constexpr float kRescaleThresh = 0.f;  // log2 units
constexpr int kPartStride = kHd + 4;   // per-row partial: O[128], m, l (+2 pad: 16-byte rows)
constexpr int kMaxSplits = 8;

struct TcSmemHdr {
  uint64_t bar_s, bar_o;
  uint32_t tmem;
  int maxlen;
  int dlen[kTcRows];
  int seg[kTcRows + 1];
  float red[2][kTcRows];  // per-half row max / final row sum exchange
  int last;               // key split: this CTA arrived last and merges
  int maxanc;             // longest ancestor list of the CTA's tokens
};
// dynamic smem: [3 KB header][Q 32 KB][K 2 x 16 KB][V 2 x 16 KB][ancestor slots]
constexpr int kTcQOff = 3072, kTcKOff = kTcQOff + 32768, kTcVOff = kTcKOff + 32768, kTcAncOff = kTcVOff + 32768;

SX_DEV uint32_t sw128(int row, int chunk) {  // byte offset of 16-byte chunk (0..7) of a 128-byte row
  return row * 128 + ((chunk ^ (row & 7)) << 4);
}
SX_DEV uint64_t desc_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
SX_DEV void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
SX_DEV float ex2_approx(float x) {  // MUFU.EX2 without the denormal fix-ups of exp2f; ex2(-inf) = +0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
SX_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// 32 consecutive fp32 columns of this thread's TMEM lane, waited in the same asm block
SX_DEV void tmem_ld32_wait(uint32_t taddr, float (&v)[32]) {
  uint32_t (&r)[32] = reinterpret_cast<uint32_t (&)[32]>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
// 64 consecutive fp32 columns of this thread's TMEM lane, waited in the same asm block
SX_DEV void tmem_ld64_wait(uint32_t taddr, float (&v)[64]) {
  uint32_t (&r)[64] = reinterpret_cast<uint32_t (&)[64]>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, "
      "%32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, "
      "%48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
        "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
        "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr)
      : "memory");
}


// Key-split bookkeeping (tcgen05 kernel, gridDim.z > 1). Every CTA of a
// (q tile, KV head) counts its arrival; the last one merges the partials of the
// working splits and resets the counter for the next launch (no second kernel).
SX_DEV bool split_arrive(const AttnArgs& a, TcSmemHdr& hd, int kvh, int zsplit) {
  int* cnt = a.counters + (long long)blockIdx.x * gridDim.y + kvh;
  __threadfence();  // this CTA's partial rows visible device-wide before the count
  __syncthreads();
  if (threadIdx.x == 0) {
    const int old = atomicAdd(cnt, 1);
    hd.last = old == zsplit - 1;
    if (hd.last) *cnt = 0;
  }
  __syncthreads();
  if (hd.last) __threadfence();
  return hd.last;
}

// O = sum_s 2^(m_s - M) O_s / sum_s 2^(m_s - M) l_s, M = max over splits that saw
// a key of the row; two threads per row, one per 64-dim half.
SX_DEV void merge_splits(const AttnArgs& a, TcSmemHdr& hd, int kvh, int zsplit, int nsplit) {
  const int tid = threadIdx.x, r = tid & (kTcRows - 1), half = tid >> 7;
  const int t = blockIdx.x * a.QB + r / a.G;
  if (t >= a.N) return;
  const float* base = a.part + (((long long)blockIdx.x * gridDim.y + kvh) * zsplit * kTcRows + r) * kPartStride;
  const long long sstride = (long long)kTcRows * kPartStride;
  float M = -1e30f;
  for (int s = 0; s < nsplit; ++s) {
    const volatile float* ps = base + s * sstride;
    if (ps[kHd + 1] > 0.f) M = fmaxf(M, ps[kHd]);
  }
  float acc[64];
#pragma unroll
  for (int j = 0; j < 64; ++j) acc[j] = 0.f;
  float L = 0.f;
  for (int s = 0; s < nsplit; ++s) {
    const float* ps = base + s * sstride;
    const float l_s = __ldcg(ps + kHd + 1);
    if (!(l_s > 0.f)) continue;  // no key of this row in the split
    const float w = exp2f(__ldcg(ps + kHd) - M);
    L += w * l_s;
    const float4* o4 = reinterpret_cast<const float4*>(ps + half * 64);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float4 v = __ldcg(o4 + j);
      acc[4 * j] += w * v.x;
      acc[4 * j + 1] += w * v.y;
      acc[4 * j + 2] += w * v.z;
      acc[4 * j + 3] += w * v.w;
    }
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  __nv_bfloat16* dst = a.out + ((long long)t * a.H + kvh * a.G + r % a.G) * kHd + half * 64;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    uint32_t w4[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) w4[j] = pack_bf16(acc[c * 8 + 2 * j] * inv, acc[c * 8 + 2 * j + 1] * inv);
    reinterpret_cast<uint4*>(dst)[c] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
  }
}

// SX_ATTN_ANC_CUDA=0: ancestors always as masked key tiles (A/B)
__constant__ int g_attn_anc_cuda = 1;

// dot of 8 bf16 pairs (16 B of a K row and 16 B of the Q row), fp32 FMA chain
SX_DEV float dot_bf16x8(const uint4& x, const uint4& y, float acc) {
  const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&x);
  const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 fa = __bfloat1622float2(a2[i]), fb = __bfloat1622float2(b2[i]);
    acc = fmaf(fa.x, fb.x, acc);
    acc = fmaf(fa.y, fb.y, acc);
  }
  return acc;
}

// Per-row ancestor keys on the CUDA cores (MHA-like groups, G <= 2, when the
// CTA's concatenated ancestor lists would add whole masked key tiles: 128 MHA
// tokens x 2-3 ancestors = 4-6 tiles of which each row uses 2-3 keys; measured
// 118.7 -> 51.4 us at N = 1024, 17 ancestors. For GQA (16 tokens x 8 heads per
// CTA) the masked tiles are few and the tensor cores win: 59.9 vs 80.0 us). Called after the
// dense tiles, with O final in TMEM: S_j = q . k_j for the row's own <= maxanc
// slots (the two column-half threads of a row each dot 64 dims, exchanged
// through the free K buffers), one max update, then O = O * 2^(m - m') +
// sum_j 2^(s_j - m') v_j chunk by chunk through TMEM. Returns the row's new
// running max; `l` (this half's share of the row sum) is rescaled and half 0
// adds the ancestors' weights.
SX_DEV float tc_ancestor_pass(const AttnArgs& a, TcSmemHdr& hd, uint8_t* base, const int* aslot,
                              const __nv_bfloat16* kbase, const __nv_bfloat16* vbase, uint32_t t_o, uint32_t lane_off,
                              int r, int half, bool o_valid, float m_used, float& l) {
  float* dots = reinterpret_cast<float*>(base + kTcKOff);  // [2][kTcRows][maxanc] partial dots
  const int A = hd.maxanc;
  const int tok = r / a.G;
  const int s0 = hd.seg[tok], na = hd.seg[tok + 1] - s0;
  uint4 qv[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) qv[c] = *reinterpret_cast<const uint4*>(base + kTcQOff + half * 16384 + sw128(r, c));
  for (int j = 0; j < na; ++j) {
    const uint4* kp = reinterpret_cast<const uint4*>(kbase + (long long)aslot[s0 + j] * kHd + half * 64);
    float d = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) d = dot_bf16x8(__ldg(kp + c), qv[c], d);
    dots[(half * kTcRows + r) * A + j] = d;
  }
  __syncthreads();
  const float scale = a.scale_log2;
  float mx = m_used;
  for (int j = 0; j < na; ++j) mx = fmaxf(mx, (dots[r * A + j] + dots[(kTcRows + r) * A + j]) * scale);
  const float f0 = o_valid ? exp2f(m_used - mx) : 0.f;
  l *= f0;
  float psum = 0.f;
#pragma unroll 1
  for (int c4 = 0; c4 < 4; ++c4) {
    float o[16];
    if (o_valid) {
      uint32_t u[16];
      tmem_ld16(t_o + lane_off + half * 64 + c4 * 16, u);
      tmem_ld_wait();
#pragma unroll
      for (int k = 0; k < 16; ++k) o[k] = __uint_as_float(u[k]) * f0;
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) o[k] = 0.f;
    }
    for (int j = 0; j < na; ++j) {
      const float p = exp2f((dots[r * A + j] + dots[(kTcRows + r) * A + j]) * scale - mx);
      if (c4 == 0) psum += p;
      const uint4* vp = reinterpret_cast<const uint4*>(vbase + (long long)aslot[s0 + j] * kHd + half * 64 + c4 * 16);
      const uint4 v0 = __ldg(vp), v1 = __ldg(vp + 1);
      const __nv_bfloat162* w0 = reinterpret_cast<const __nv_bfloat162*>(&v0);
      const __nv_bfloat162* w1 = reinterpret_cast<const __nv_bfloat162*>(&v1);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 x0 = __bfloat1622float2(w0[k]), x1 = __bfloat1622float2(w1[k]);
        o[2 * k] = fmaf(p, x0.x, o[2 * k]);
        o[2 * k + 1] = fmaf(p, x0.y, o[2 * k + 1]);
        o[8 + 2 * k] = fmaf(p, x1.x, o[8 + 2 * k]);
        o[8 + 2 * k + 1] = fmaf(p, x1.y, o[8 + 2 * k + 1]);
      }
    }
    uint32_t u[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) u[k] = __float_as_uint(o[k]);
    tmem_st16(t_o + lane_off + half * 64 + c4 * 16, u);
  }
  tmem_st_wait();
  if (half == 0) l += psum;
  return mx;
}

__global__ void __launch_bounds__(kTcThreads, 2) tree_attention_tc_kernel(const AttnArgs a) {
  griddep_launch_dependents();
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  TcSmemHdr& hd = *reinterpret_cast<TcSmemHdr*>(base);
  int* aslot = reinterpret_cast<int*>(base + kTcAncOff);
  const uint32_t qs = smem_u32(base + kTcQOff), ks0 = smem_u32(base + kTcKOff), vs0 = smem_u32(base + kTcVOff);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int kvh = blockIdx.y;
  const int t0 = blockIdx.x * a.QB;
  const __nv_bfloat16* kbase = a.kc + (long long)kvh * a.slots * kHd;
  const __nv_bfloat16* vbase = a.vc + (long long)kvh * a.slots * kHd;

  if (tid == 0) {
    hd.maxlen = 0;
    mbar_init(&hd.bar_s, 1);
    mbar_init(&hd.bar_o, 1);
    fence_barrier_init();
  }
  // Q first (its own cp.async group): the load overlaps the per-token metadata below.
  // Row r = token-major, head-minor; 16-byte chunk c of the row -> region c / 8.
  for (int i = tid; i < kTcRows * 16; i += kTcThreads) {
    const int r = i >> 4, c = i & 15;
    const int t = t0 + r / a.G, h = kvh * a.G + r % a.G;
    const __nv_bfloat16* src = a.q + ((long long)(t < a.N ? t : 0) * a.H + h) * kHd + c * 8;
    cp_async16(qs + (c >> 3) * 16384 + sw128(r, c & 7), src, t < a.N ? 16 : 0);
  }
  cp_async_commit();
  __syncthreads();
  if (tid < kTcRows) {
    const int t = t0 + tid / a.G;
    const int dl = t < a.N ? (a.dense_len ? a.dense_len[t] : a.dense_const) : 0;
    hd.dlen[tid] = dl;
    atomicMax(&hd.maxlen, dl);
  }
  if (tid < a.QB) {
    const int t = t0 + tid;
    hd.seg[tid + 1] = (t < a.N && a.anc_len) ? a.anc_len[t] : 0;
  }
  __syncthreads();
  if (tid == 0) {
    hd.seg[0] = 0;
    for (int i = 1; i <= a.QB; ++i) hd.seg[i] += hd.seg[i - 1];
  }
  __syncthreads();
  const int n_anc = hd.seg[a.QB];
  if (tid == 0) {
    int mx = 0;
    for (int i = 0; i < a.QB; ++i) mx = max(mx, hd.seg[i + 1] - hd.seg[i]);
    hd.maxanc = mx;
  }
  for (int i = tid; i < a.QB * a.A; i += kTcThreads) {
    const int tl = i / a.A, j = i % a.A, t = t0 + tl;
    if (t < a.N && j < hd.seg[tl + 1] - hd.seg[tl]) aslot[hd.seg[tl] + j] = a.anc_base + a.anc[(long long)t * a.A + j];
  }
  __syncthreads();  // aslot visible to the K/V loaders
  static_assert(sizeof(TcSmemHdr) <= kTcQOff, "attention smem header overlaps Q");
  const int maxlen = hd.maxlen;
  // ancestors on the CUDA cores when they would add whole masked key tiles
  // (unsplit launches; a row's list <= 32 keys so its dots fit the K buffers)
  const bool anc_cuda = g_attn_anc_cuda && a.G <= 2 && gridDim.z == 1 && hd.maxanc <= 32 &&
                        (maxlen + n_anc + kKeyTile - 1) / kKeyTile > (maxlen + kKeyTile - 1) / kKeyTile;
  const int n_anc_keys = anc_cuda ? 0 : n_anc;
  const int ntiles_all = (maxlen + n_anc_keys + kKeyTile - 1) / kKeyTile;
  // key split (gridDim.z > 1): the first `nsplit` of the launched splits take
  // >= 4 key tiles each (fewer splits for short contexts -- a split costs a
  // CTA prologue and a partial round trip); this CTA takes tiles [kt0, kt0 + ntiles)
  const int zsplit = gridDim.z, split = blockIdx.z;
  const int nsplit = zsplit > 1 ? max(1, min(zsplit, ntiles_all / 4)) : 1;
  if (split >= nsplit) {  // idle split: no TMEM, no partial -- only the arrival count
    cp_async_wait<0>();
    if (split_arrive(a, hd, kvh, zsplit) && nsplit > 1) merge_splits(a, hd, kvh, zsplit, nsplit);
    return;
  }
  const int kt0 = (int)(((long long)ntiles_all * split) / nsplit);
  const int ntiles = (int)(((long long)ntiles_all * (split + 1)) / nsplit) - kt0;
  if (warp == 0) tmem_alloc(&hd.tmem, kTcTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  // thread: 16-byte chunk c of key rows r0, r0 + 16, r0 + 32, r0 + 48 (same swizzle phase)
  const int lc = tid & 15, lr0 = tid >> 4;
  const uint32_t loff = (lc >> 3) * 8192 + sw128(lr0, lc & 7);
  auto load_kv = [&](int tile, int local) {
    const int buf = local & 1;
    const uint32_t kd = ks0 + buf * 16384 + loff, vd = vs0 + buf * 16384 + loff;
#pragma unroll
    for (int k = 0; k < kKeyTile * 16 / kTcThreads; ++k) {
      const int key = tile * kKeyTile + lr0 + (kTcThreads / 16) * k;
      int slot = key;
      bool ok = true;
      if (key >= maxlen) {
        const int j = key - maxlen;
        ok = j < n_anc_keys;
        slot = ok ? aslot[j] : 0;
      }
      const long long off = (long long)slot * kHd + lc * 8;
      cp_async16(kd + k * (kTcThreads / 16) * 128, kbase + off, ok ? 16 : 0);
      cp_async16(vd + k * (kTcThreads / 16) * 128, vbase + off, ok ? 16 : 0);
    }
  };
  if (ntiles > 0) load_kv(kt0, 0);
  cp_async_commit();  // group: tile 0
  if (ntiles > 1) load_kv(kt0 + 1, 1);
  cp_async_commit();  // group: tile 1 (possibly empty)

  const uint32_t tmem = hd.tmem;
  const uint32_t t_s = tmem, t_o = tmem + 64;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;  // TMEM lane quadrant = warp % 4
  const int r = tid & (kTcRows - 1), half = tid >> 7;  // row, column half (keys / O dims)
  const int dl = hd.dlen[r];
  const int slo = anc_cuda ? 0x3fffffff : maxlen + hd.seg[r / a.G];
  const int shi = anc_cuda ? 0x3fffffff : maxlen + hd.seg[r / a.G + 1];
  constexpr uint32_t idesc_s = idesc_bf16_f32(kTcRows, kKeyTile);
  constexpr uint32_t idesc_o = idesc_bf16_f32(kTcRows, kHd) | (1u << 16);  // B (V) MN-major
  float m_used = -1e30f, l = 0.f;
  const float scale = a.scale_log2;

  for (int i = 0; i < ntiles; ++i) {
    const int kt = kt0 + i, buf = i & 1;
    const uint32_t kb = ks0 + buf * 16384, vb = vs0 + buf * 16384;
    if (i == 0) cp_async_wait<1>();
    else cp_async_wait<0>();
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {  // S = Q K^T
      tc_fence_after();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint64_t da = desc_sw128(qs + (j >> 2) * 16384 + (j & 3) * 32, 16, 1024);
        const uint64_t db = desc_sw128(kb + (j >> 2) * 8192 + (j & 3) * 32, 16, 1024);
        tc_mma_bf16(t_s, da, db, idesc_s, j > 0);
      }
      tc_commit(&hd.bar_s);
    }
    if (i >= 1) {  // P V of the previous tile done: its K (holding P) and V buffers are free
      mbar_wait(&hd.bar_o, (i - 1) & 1);
      if (i + 1 < ntiles) load_kv(kt + 1, i + 1);
      cp_async_commit();
    }
    mbar_wait(&hd.bar_s, i & 1);
    tc_fence_after();
    float sv[32];
    tmem_ld32_wait(t_s + lane_off + half * 32, sv);
    // mask + scale (branch-free: key < dl, or key in the row's own ancestor segment), partial max
    const int kbase_i = kt * kKeyTile + half * 32;
    const int dlr = dl - kbase_i, slr = slo - kbase_i, shr = shi - kbase_i;
    float pm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const bool ok = (j < dlr) | ((j >= slr) & (j < shr));
      sv[j] = ok ? sv[j] * scale : -INFINITY;
      pm[j & 3] = fmaxf(pm[j & 3], sv[j]);
    }
    hd.red[half][r] = fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3]));
    __syncthreads();
    const float mx = fmaxf(hd.red[0][r], hd.red[1][r]);  // identical in both halves
    const bool move = mx > m_used + a.rescale_thresh;
    const float m_new = move ? mx : m_used;
    const float factor = move ? exp2f(m_used - m_new) : 1.f;
    l *= factor;
    m_used = m_new;
    if (__any_sync(0xffffffff, move) && i > 0) {  // warp-collective TMEM round trip over this half of O
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t u[16];
        const uint32_t ta = t_o + lane_off + half * 64 + c * 16;
        tmem_ld16(ta, u);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) u[j] = __float_as_uint(__uint_as_float(u[j]) * factor);
        tmem_st16(ta, u);
      }
      tmem_st_wait();
    }
    // P (this half's 32 keys = 16-byte chunks 4*half .. 4*half+3 of row r) -> the K buffer of this tile
    uint8_t* prow = base + kTcKOff + buf * 16384;
    float ps[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t w[4];
      float s8 = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float p0 = ex2_approx(sv[c * 8 + 2 * j] - m_used), p1 = ex2_approx(sv[c * 8 + 2 * j + 1] - m_used);
        s8 += p0 + p1;
        w[j] = pack_bf16(p0, p1);
      }
      ps[c] = s8;
      *reinterpret_cast<uint4*>(prow + sw128(r, half * 4 + c)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    l += (ps[0] + ps[1]) + (ps[2] + ps[3]);  // this half's share of the row sum
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {  // O += P V
      tc_fence_after();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t da = desc_sw128(kb + j * 32, 16, 1024);
        const uint64_t db = desc_sw128(vb + j * 2048, 8192, 1024);
        tc_mma_bf16(t_o, da, db, idesc_o, i > 0 || j > 0);
      }
      tc_commit(&hd.bar_o);
    }
  }
  // epilogue: O / l -> bf16; each thread stores its half (64 dims) of row r.
  // Key split: the unnormalised O half, plus (m, l) of the row, go to the
  // workspace instead and attn_combine_kernel merges the splits.
  if (ntiles > 0) {
    mbar_wait(&hd.bar_o, (ntiles - 1) & 1);
    tc_fence_after();
  }
  bool o_valid = ntiles > 0;
  if (anc_cuda) {
    m_used = tc_ancestor_pass(a, hd, base, aslot, kbase, vbase, t_o, lane_off, r, half, o_valid, m_used, l);
    o_valid = true;
  }
  hd.red[half][r] = l;
  __syncthreads();
  const float lt = hd.red[0][r] + hd.red[1][r];
  const int t = t0 + r / a.G;
  float* prow_ws = nullptr;
  if (nsplit > 1) {
    prow_ws = a.part + ((((long long)blockIdx.x * gridDim.y + kvh) * zsplit + split) * kTcRows + r) * kPartStride;
    if (half == 0) {
      prow_ws[kHd] = m_used;
      prow_ws[kHd + 1] = lt;
    }
  }
  __nv_bfloat16* dst = a.out + ((long long)t * a.H + kvh * a.G + r % a.G) * kHd + half * 64;
  const float inv = lt > 0.f ? 1.f / lt : 0.f;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t u[16];
    if (o_valid) {
      tmem_ld16(t_o + lane_off + half * 64 + c * 16, u);
      tmem_ld_wait();
    }
    if (prow_ws) {
      float4* d4 = reinterpret_cast<float4*>(prow_ws + half * 64 + c * 16);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        d4[j] = o_valid ? make_float4(__uint_as_float(u[4 * j]), __uint_as_float(u[4 * j + 1]),
                                         __uint_as_float(u[4 * j + 2]), __uint_as_float(u[4 * j + 3]))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
      continue;
    }
    uint32_t w[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      w[j] = o_valid ? pack_bf16(__uint_as_float(u[2 * j]) * inv, __uint_as_float(u[2 * j + 1]) * inv) : 0u;
    if (t < a.N) {
      uint4* d4 = reinterpret_cast<uint4*>(dst + c * 16);
      d4[0] = make_uint4(w[0], w[1], w[2], w[3]);
      d4[1] = make_uint4(w[4], w[5], w[6], w[7]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kTcTmemCols);
  if (zsplit > 1 && split_arrive(a, hd, kvh, zsplit) && nsplit > 1) merge_splits(a, hd, kvh, zsplit, nsplit);
}



static int g_attn_impl = 0;  // 0 by shape, 1 mma.sync only, 2 tcgen05 only

}  // namespace sx

using namespace sx;

// key splits of the tcgen05 kernel for a grid of `ctas` CTAs: enough to put
// ~2 CTAs on every SM when the grid alone cannot
static int attn_splits(long long ctas) {
  if (ctas >= 148) return 1;
  const long long s = (2 * 148 + ctas - 1) / ctas;
  return (int)(s < kMaxSplits ? s : kMaxSplits);
}

// Workspace = [fixed arrival-counter header][partials]. The header size does not
// depend on N: callers reuse one zero-once workspace across launches of every
// shape (draft buckets, one-token graphs, target passes), and a counter slot must
// never alias partials a differently-sized launch wrote. Splits happen only for
// grids of < 148 CTAs, so 148 counters always fit.
constexpr long long kAttnCounterBytes = 1024;
static_assert(148 * 4 <= kAttnCounterBytes, "counter header too small");

extern "C" long long sx_tree_attention_ws_bytes(int N, int H, int KVH) {
  if (N <= 0 || KVH <= 0 || H % KVH || kTcRows % (H / KVH)) return 0;
  const int qb = kTcRows / (H / KVH);
  const long long ctas = (long long)((N + qb - 1) / qb) * KVH;
  const int S = attn_splits(ctas);
  // the counters must be zero on first use; the kernel resets them after each launch
  return S > 1 ? kAttnCounterBytes + ctas * S * kTcRows * kPartStride * (long long)sizeof(float) : 0;
}

extern "C" int sx_tree_attention_ws(const void* q, const void* kcache, const void* vcache, long long slots,
                                    const int* dense_len, int dense_const, const int* anc, int anc_base,
                                    const int* anc_len, int A, void* out, int N, int H, int KVH, void* ws,
                                    long long ws_bytes, cudaStream_t stream) {
  if (N <= 0) return SX_OK;
  if (KVH <= 0 || H % KVH) return arg_error("attention: H (%d) must be a multiple of KVH (%d)", H, KVH);
  const int G = H / KVH;
  if (G > kAttRows || kAttRows % G) return arg_error("attention: group size %d must divide %d", G, kAttRows);
  if (A < 0) return arg_error("attention: negative ancestor width %d", A);
  AttnArgs a;
  a.q = reinterpret_cast<const __nv_bfloat16*>(q);
  a.kc = reinterpret_cast<const __nv_bfloat16*>(kcache);
  a.vc = reinterpret_cast<const __nv_bfloat16*>(vcache);
  a.slots = slots;
  a.dense_len = dense_len;
  a.dense_const = dense_const;
  a.anc_base = anc_base;
  a.anc = anc;
  a.anc_len = anc_len;
  a.A = A;
  a.out = reinterpret_cast<__nv_bfloat16*>(out);
  a.N = N;
  a.H = H;
  a.KVH = KVH;
  a.G = G;
  a.QB = kAttRows / G;
  a.scale_log2 = 1.4426950408889634f / sqrtf((float)kHd);
  a.rescale_thresh = kRescaleThresh;
  a.splits = 1;
  a.part = nullptr;
  a.counters = nullptr;
  // Kernel choice (tools/attn_probe.py): the tcgen05 kernel, with its key tiles
  // split over up to 8 CTAs when the grid is smaller than the machine (needs the
  // workspace, sx_tree_attention_ws_bytes). Narrow groups (G < 4) on mid-size
  // batches (128 < N, < 148 CTAs; 64 < N without a workspace) take the 64-row
  // mma.sync loop: each tcgen05 CTA would carry 128 tokens' ancestor lists.
  const int tc_qb = kTcRows % G ? 0 : kTcRows / G;
  const long long tc_ctas = tc_qb ? (long long)((N + tc_qb - 1) / tc_qb) * KVH : 0;
  const long long need = sx_tree_attention_ws_bytes(N, H, KVH);
  const bool split_ok = need > 0 && ws != nullptr && ws_bytes >= need;
  const bool mma_fits = (long long)(kAttRows / G) * A <= kMaxAncKeys;  // its static ancestor list
  const bool mma_wins = G < 4 && N > (split_ok ? 128 : 64) && tc_ctas < 148;
  const bool use_tc = g_attn_impl == 0 && tc_qb > 0 && (!mma_wins || !mma_fits);
  if (use_tc || g_attn_impl == 2) {
    if (kTcRows % G) return arg_error("attention: group size %d must divide %d", G, kTcRows);
    a.QB = kTcRows / G;
    const long long anc_bytes = 4LL * a.QB * (A > 0 ? A : 0);
    if (anc_bytes > 64 * 1024)
      return arg_error("attention: %d tokens x %d ancestors exceed the per-CTA ancestor list", a.QB, A);
    if (split_ok) {
      a.splits = attn_splits(tc_ctas);
      a.counters = reinterpret_cast<int*>(ws);
      a.part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + kAttnCounterBytes);
    }
    static const int anc_cuda_init = [] {
      const int v = getenv("SX_ATTN_ANC_CUDA") ? atoi(getenv("SX_ATTN_ANC_CUDA")) : 1;
      if (v != 1) cudaMemcpyToSymbol(g_attn_anc_cuda, &v, sizeof(int));
      return v;
    }();
    (void)anc_cuda_init;
    const size_t smem = 1024 + kTcAncOff + (size_t)((anc_bytes + 15) & ~15LL);
    if (int st = ensure_smem_attr((const void*)tree_attention_tc_kernel, (int)smem)) return st;
    dim3 grid((N + a.QB - 1) / a.QB, KVH, a.splits);
    tree_attention_tc_kernel<<<grid, kTcThreads, smem, stream>>>(a);
    SX_CHECK_LAUNCH("tree_attention_tc_kernel");
    return SX_OK;
  }
  if ((long long)(kAttRows / G) * A > kMaxAncKeys)
    return arg_error("attention: %d tokens x %d ancestors exceed %d ancestor keys per CTA", kAttRows / G, A, kMaxAncKeys);
  const size_t smem = sizeof(AttnSmem);
  if (int st = ensure_smem_attr((const void*)tree_attention_kernel, (int)smem)) return st;
  dim3 grid((N + a.QB - 1) / a.QB, KVH);
  tree_attention_kernel<<<grid, kAttWarps * 32, smem, stream>>>(a);
  SX_CHECK_LAUNCH("tree_attention_kernel");
  return SX_OK;
}

extern "C" int sx_tree_attention(const void* q, const void* kcache, const void* vcache, long long slots,
                                 const int* dense_len, int dense_const, const int* anc, int anc_base,
                                 const int* anc_len, int A, void* out, int N, int H, int KVH, cudaStream_t stream) {
  return sx_tree_attention_ws(q, kcache, vcache, slots, dense_len, dense_const, anc, anc_base, anc_len, A, out, N, H,
                              KVH, nullptr, 0, stream);
}

extern "C" int sx_attention_set_impl(int impl) {
  if (impl < 0 || impl > 2) return arg_error("attention impl %d (0 by shape, 1 mma.sync, 2 tcgen05)", impl);
  g_attn_impl = impl;
  return SX_OK;
}
