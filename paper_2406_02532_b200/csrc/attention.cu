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
// One flash-attention main loop on tensor cores (bf16 mma.sync m16n8k16, fp32
// online softmax, cp.async double-buffered K/V tiles, XOR-swizzled shared
// memory) covers both parts in one key space: the committed prefix [0, maxlen)
// followed by the ancestor keys gathered by slot -- the concatenated ancestor
// lists of the CTA's tokens (<= D+1 keys each), each row masked to its own
// segment -- so the ancestors fill the last partial committed tile. GQA:
// one CTA serves one KV head and 64 query rows = (64 / G) tokens x G heads.
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

}  // namespace sx

using namespace sx;

extern "C" int sx_tree_attention(const void* q, const void* kcache, const void* vcache, long long slots,
                                 const int* dense_len, int dense_const, const int* anc, int anc_base,
                                 const int* anc_len, int A, void* out, int N, int H, int KVH, cudaStream_t stream) {
  if (N <= 0) return SX_OK;
  if (KVH <= 0 || H % KVH) return arg_error("attention: H (%d) must be a multiple of KVH (%d)", H, KVH);
  const int G = H / KVH;
  if (G > kAttRows || kAttRows % G) return arg_error("attention: group size %d must divide %d", G, kAttRows);
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
  if (A < 0 || (long long)(kAttRows / G) * A > kMaxAncKeys)
    return arg_error("attention: %d tokens x %d ancestors exceed %d ancestor keys per CTA", kAttRows / G, A, kMaxAncKeys);
  const size_t smem = sizeof(AttnSmem);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tree_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid((N + a.QB - 1) / a.QB, KVH);
  tree_attention_kernel<<<grid, kAttWarps * 32, smem, stream>>>(a);
  SX_CHECK_LAUNCH("tree_attention_kernel");
  return SX_OK;
}
