"""Llama-shaped draft / target models on the B200 (device models for the engine).

A `LlamaModel` is a `LanguageModel` plugin (pkg/src/speckit/models.py:32-63)
whose forward runs entirely in hand-written sm_100a kernels through the C ABI:
tcgen05 GEMMs for every projection (fused SwiGLU and residual epilogues),
tree-masked attention with an explicit ancestor list per query, RMSNorm /
RoPE / KV scatter, and the fp32 LM head. PyTorch only allocates memory.

It keeps a KV cache and a prefix cache keyed by token ids ("committed" tokens
whose KV sits in slots 0..c-1 at positions equal to their slots), so the
stateless reference API -- next_distribution(prefix) -- and the engine's
`precompute(prefix, ...)` reuse everything already computed for a shared
prefix. After each walk, `commit_walk` moves the KV rows of the accepted path
into the committed region (kv_compact); the draft also keeps the KV of every
node it expanded while building the tree.

Weights are random-init (N(0, std), RMSNorm = 1, untied) from a seed, in the
named architecture's shapes; an optional *synthetic* prev-token bias (a shared
low-rank table added to the logits of draft and target alike) and a logit scale
make draft and target agree like a trained pair; it is off by
default and always reported when on.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Sequence

import numpy as np
import torch

from . import _lib
from . import kernels as K
from .models import LanguageModel, _WS, _check_prefix
from .tp import TPShard, gather_vocab
from .tree import BuilderParams, tree_tables


@dataclass(frozen=True)
class LlamaConfig:
    vocab: int
    d: int
    layers: int
    heads: int
    kv_heads: int
    ff: int
    rope_theta: float = 10000.0
    eps: float = 1e-5
    head_dim: int = 128
    name: str = "llama"

    @property
    def qkv_out(self) -> int:
        return (self.heads + 2 * self.kv_heads) * self.head_dim

    def n_params(self) -> int:
        per_layer = self.qkv_out * self.d + self.d * self.heads * self.head_dim + 3 * self.d * self.ff + 2 * self.d
        return self.layers * per_layer + 2 * self.vocab * self.d + self.d

    def weight_bytes(self) -> int:
        return 2 * self.n_params()

    def kv_bytes_per_slot(self) -> int:
        return self.layers * 2 * self.kv_heads * self.head_dim * 2


PRESETS = {
    "llama2-7b": LlamaConfig(32000, 4096, 32, 32, 32, 11008, 1e4, 1e-5, name="llama2-7b"),
    "llama2-70b": LlamaConfig(32000, 8192, 80, 64, 8, 28672, 1e4, 1e-5, name="llama2-70b"),
    "llama3-8b": LlamaConfig(128256, 4096, 32, 32, 8, 14336, 5e5, 1e-5, name="llama3-8b"),
    "llama3-70b": LlamaConfig(128256, 8192, 80, 64, 8, 28672, 5e5, 1e-5, name="llama3-70b"),
    # demo-sized (BASELINE config 1 restated): d=256, 4 layers, V=32000
    "tiny": LlamaConfig(32000, 256, 4, 2, 1, 704, 1e4, 1e-5, name="tiny"),
    "tiny-draft": LlamaConfig(32000, 256, 2, 2, 2, 512, 1e4, 1e-5, name="tiny-draft"),
}


@dataclass
class SyntheticBias:
    """Shared prev-token logit bias (low rank): logits[t] += scale * U[x_t] . W."""

    seed: int = 1234
    rank: int = 64
    scale: float = 1.0


def _rope_tables(cfg: LlamaConfig, max_pos: int, device) -> tuple[torch.Tensor, torch.Tensor]:
    # HF Llama convention, computed in fp32
    inv_freq = 1.0 / (cfg.rope_theta ** (torch.arange(0, cfg.head_dim, 2, dtype=torch.int64).float() / cfg.head_dim))
    t = torch.arange(max_pos, dtype=torch.int64).float()
    freqs = torch.outer(t, inv_freq)
    return freqs.cos().contiguous().to(device), freqs.sin().contiguous().to(device)


def interleave_gate_up(gate: torch.Tensor, up: torch.Tensor) -> torch.Tensor:
    """[gate; up] interleaved in 64-row blocks -- the stored layout of the
    SwiGLU projection: one GEMM tile of 128 weight rows covers gate and up of
    the same 64 features, so the epilogue (SX_EPI_SWIGLU_IL) writes
    silu(gate) * up without a second accumulator."""
    f, d = gate.shape
    if f % 64:
        raise ValueError(f"FFN width {f} must be a multiple of 64")
    return torch.stack([gate.reshape(f // 64, 64, d), up.reshape(f // 64, 64, d)], dim=1).reshape(2 * f, d)


def split_gate_up(wgu: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    f2, d = wgu.shape
    v = wgu.reshape(f2 // 128, 2, 64, d)
    return v[:, 0].reshape(f2 // 2, d), v[:, 1].reshape(f2 // 2, d)


def layer_layout(cfg: LlamaConfig, shard: TPShard | None = None,
                 stored: bool = True, elem: int = 2) -> tuple[dict[str, tuple[int, tuple[int, ...]]], int]:
    """Byte offsets of one decoder layer's tensors in a contiguous buffer
    (256-B aligned, the unit streamed in offload mode); `shard`: this rank's
    tensor-parallel slice of the layer (tp.py). stored=True: the HBM layout
    (gate/up interleaved as "wgu"); False: the draw layout (wg, wu apart).
    elem: bytes per element (2 = bf16, 4 = the fp32 target mode)."""
    shapes = dict((TPShard(0, 1) if shard is None else shard).local_shapes(cfg))
    if stored:
        f, d = shapes.pop("wg")
        shapes.pop("wu")
        wd = shapes.pop("wd")
        n1, n2 = shapes.pop("n1"), shapes.pop("n2")
        shapes.update({"wgu": (2 * f, d), "wd": wd, "n1": n1, "n2": n2})
    out, off = {}, 0
    for k, shp in shapes.items():
        out[k] = (off, shp)
        off += (math.prod(shp) * elem + 255) // 256 * 256
    return out, off


def layer_views(buf: torch.Tensor, layout, dtype: torch.dtype = torch.bfloat16) -> dict[str, torch.Tensor]:
    e = torch.empty((), dtype=dtype).element_size()
    return {k: buf[o : o + math.prod(s) * e].view(dtype).view(s) for k, (o, s) in layout.items()}


class LlamaWeights:
    """bf16 weights in nn.Linear layout ([out, in]); each decoder layer is one
    contiguous buffer -- in HBM, or (offload) in pinned host memory. Gate and
    up projections are stored interleaved ("wgu", interleave_gate_up)."""

    def __init__(self, cfg: LlamaConfig, seed: int, device, std: float = 0.02, lm_scale: float = 1.0,
                 offload: bool = False, shard: TPShard | None = None, init: str = "device",
                 dtype: torch.dtype = torch.bfloat16):
        """init="device": drawn by a CUDA generator (fast at 70B); "host": drawn
        by a CPU generator and uploaded -- the same values `host_weights_fp32`
        draws without a GPU (the CPU reference arm's copy of small models)."""
        if init not in ("device", "host"):
            raise ValueError(f"init must be 'device' or 'host', got {init!r}")
        self.cfg = cfg
        self.offload = offload
        self.shard = shard
        self.dtype = dtype
        elem = torch.empty((), dtype=dtype).element_size()
        host_draw = init == "host"
        g = torch.Generator(device="cpu" if host_draw else device)
        g.manual_seed(seed)

        def rnd_(t, s=std):
            if host_draw:
                return t.copy_(torch.empty(t.shape, dtype=t.dtype).normal_(0.0, s, generator=g))
            return t.normal_(0.0, s, generator=g)

        self.emb = rnd_(torch.empty((cfg.vocab, cfg.d), dtype=dtype, device=device))
        self.layout, self.layer_bytes = layer_layout(cfg, shard, elem=elem)
        self.layer_bufs: list[torch.Tensor] = []
        self.layers = []
        tmp = torch.empty(self.layer_bytes, dtype=torch.uint8, device=device) if offload else None
        # every layer is drawn in the full, unsharded draw layout (same draw order
        # for every TP degree / storage layout), then sliced (TP) and stored
        gen_layout, gen_bytes = layer_layout(cfg, stored=False, elem=elem)
        gen_tmp = torch.empty(gen_bytes, dtype=torch.uint8, device=device)
        sh = shard if shard is not None else TPShard(0, 1)
        for _ in range(cfg.layers):
            buf = tmp if offload else torch.empty(self.layer_bytes, dtype=torch.uint8, device=device)
            v = layer_views(buf, self.layout, dtype)
            src = layer_views(gen_tmp, gen_layout, dtype)
            for k in ("wqkv", "wo", "wg", "wu", "wd"):  # draw order
                rnd_(src[k])
            for k in ("wqkv", "wo", "wd"):
                v[k].copy_(sh.shard(cfg, k, src[k]))
            v["wgu"].copy_(interleave_gate_up(sh.shard(cfg, "wg", src["wg"]), sh.shard(cfg, "wu", src["wu"])))
            v["n1"].fill_(1.0)
            v["n2"].fill_(1.0)
            if offload:
                host = torch.empty(self.layer_bytes, dtype=torch.uint8, pin_memory=True)
                host.copy_(buf)
                self.layer_bufs.append(host)
                self.layers.append(layer_views(host, self.layout, dtype))
            else:
                self.layer_bufs.append(buf)
                self.layers.append(v)
        del tmp, gen_tmp
        self.nf = torch.ones(cfg.d, dtype=dtype, device=device)
        self.lm = rnd_(torch.empty((cfg.vocab, cfg.d), dtype=dtype, device=device), std * lm_scale)
        if shard is not None:
            self.lm = shard.shard(cfg, "lm", self.lm)

    def to_cpu_fp32(self) -> dict:
        """fp32 CPU copy for the CPU reference forward (oracle/llama_ref.py)."""
        f = lambda t: t.float().cpu()  # noqa: E731

        def layer(L):
            out = {k: f(v) for k, v in L.items() if k != "wgu"}
            out["wg"], out["wu"] = (f(t) for t in split_gate_up(L["wgu"]))
            return out

        return {
            "emb": f(self.emb),
            "layers": [layer(L) for L in self.layers],
            "nf": f(self.nf),
            "lm": f(self.lm),
        }


def host_weights_fp32(cfg: LlamaConfig, seed: int, std: float = 0.02, lm_scale: float = 1.0) -> dict:
    """The weights LlamaWeights(init="host") draws -- same CPU generator, same
    draw order, bf16 values -- as fp32 CPU tensors in the CPU reference forward's
    layout (oracle/llama_ref.py). No GPU needed (bench.py's reference arm)."""
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    rnd = lambda shape, s=std: torch.empty(shape, dtype=torch.bfloat16).normal_(0.0, s, generator=g)  # noqa: E731
    emb = rnd((cfg.vocab, cfg.d)).float()
    shapes = TPShard(0, 1).local_shapes(cfg)
    layers = []
    for _ in range(cfg.layers):
        L = {k: rnd(shapes[k]).float() for k in ("wqkv", "wo", "wg", "wu", "wd")}
        L["n1"] = torch.ones(cfg.d)
        L["n2"] = torch.ones(cfg.d)
        layers.append(L)
    lm = rnd((cfg.vocab, cfg.d), std * lm_scale).float()
    return {"emb": emb, "layers": layers, "nf": torch.ones(cfg.d), "lm": lm}


class LayerStreamer:
    """Stage 3: per-layer weight streaming from pinned host RAM through a ring of
    `nbuf` HBM staging buffers (nbuf = 2 is plain double buffering).

    Copies run on a dedicated stream (copy engines) through sx_stream_copy; the
    k-th copy lands in staging buffer k % nbuf after the compute stream released
    it. Layers are issued in cyclic order, so finishing layer L-1 of one pass
    immediately starts loading layers 0..nbuf-1 of the next pass -- they stream
    in while the draft builds the next tree (the paper's prefetch); a ring deep
    enough to cover the draft phase keeps the host link busy all iteration."""

    def __init__(self, weights: LlamaWeights, device, nbuf: int = 2):
        self.w = weights
        self.L = weights.cfg.layers
        self.nbuf = nbuf
        self.stream = torch.cuda.Stream(device)
        self.bufs = [torch.empty(weights.layer_bytes, dtype=torch.uint8, device=device) for _ in range(nbuf)]
        self.views = [layer_views(b, weights.layout) for b in self.bufs]
        self.ready = [torch.cuda.Event() for _ in range(nbuf)]
        self.free = [torch.cuda.Event() for _ in range(nbuf)]
        for e in self.ready + self.free:  # materialise the event handles
            e.record(self.stream)
        self.pending: list[tuple[int, int]] = []  # (layer, buffer) copies issued, FIFO
        self.k = 0
        self.next_layer = 0
        self.bytes = 0
        torch.cuda.synchronize(device)

    def _issue(self) -> None:
        li, b = self.next_layer, self.k % self.nbuf
        _lib.call("sx_stream_copy", _lib.ptr(self.bufs[b]), self.w.layer_bufs[li].data_ptr(), self.w.layer_bytes, 1,
                  int(self.stream.cuda_stream), self.free[b].cuda_event, self.ready[b].cuda_event)
        self.pending.append((li, b))
        self.bytes += self.w.layer_bytes
        self.k += 1
        self.next_layer = (li + 1) % self.L

    def acquire(self, li: int) -> dict[str, torch.Tensor]:
        while len(self.pending) < self.nbuf:
            self._issue()
        layer, b = self.pending[0]
        if layer != li:
            raise RuntimeError(f"layer streamer out of order: expected {layer}, got {li}")
        torch.cuda.current_stream().wait_event(self.ready[b])
        return self.views[b]

    def release(self, li: int) -> None:
        _, b = self.pending.pop(0)
        self.free[b].record(torch.cuda.current_stream())
        self._issue()  # refill the freed buffer with the next layer in cyclic order


class _Buffers:
    def __init__(self, cfg: LlamaConfig, n: int, device, shard: TPShard | None = None, reduce_bf16: bool = False,
                 act_dtype: torch.dtype = torch.bfloat16):
        self.n = n
        sh = TPShard(0, 1) if shard is None else shard
        H = cfg.heads // sh.world
        KVH = cfg.kv_heads // sh.world
        self.x = torch.empty((n, cfg.d), dtype=torch.float32, device=device)
        # o / down projection output (TP: the partial sums that are all-reduced)
        self.y = torch.empty((n, cfg.d), dtype=torch.bfloat16 if reduce_bf16 else torch.float32, device=device)
        self.h = torch.empty((n, cfg.d), dtype=act_dtype, device=device)
        self.qkv = torch.empty((n, (H + 2 * KVH) * cfg.head_dim), dtype=act_dtype, device=device)
        self.q = torch.empty((n, H * cfg.head_dim), dtype=act_dtype, device=device)
        self.att = torch.empty((n, H * cfg.head_dim), dtype=act_dtype, device=device)
        self.act = torch.empty((n, cfg.ff // sh.world), dtype=act_dtype, device=device)
        self.logits = torch.empty((n, cfg.vocab), dtype=torch.float32, device=device)
        if sh.world > 1:  # vocab-parallel LM head: local slice + all-gather staging
            self.logits_l = torch.empty((n, cfg.vocab // sh.world), dtype=torch.float32, device=device)
            self.logits_g = torch.empty((sh.world, n, cfg.vocab // sh.world), dtype=torch.float32, device=device)
            self.argmax_keys = torch.empty((n, 1), dtype=torch.int64, device=device)  # KV1 (tp_argmax)
        self.tok = torch.empty(n, dtype=torch.int32, device=device)
        self.pos = torch.empty(n, dtype=torch.int32, device=device)


class LlamaModel(LanguageModel):
    """Llama-shaped model resident in HBM; a device model for the SpecExec engine."""

    backend = "llama"
    _serial = 0

    def __init__(
        self,
        cfg: LlamaConfig | str,
        seed: int = 0,
        max_ctx: int = 4096,
        max_tokens: int = 1024,
        std: float = 0.02,
        lm_scale: float = 1.0,
        synthetic: SyntheticBias | None = None,
        device=None,
        offload: bool = False,
        tp=None,
        reduce_bf16: bool = True,
        tp_fused: bool | None = None,
        tp_argmax: bool = False,
        offload_buffers: int = 8,
        init: str = "device",
        dtype: str = "bf16",
    ):
        """offload_buffers: HBM staging slots of the layer streamer (offload mode);
        beyond the 2 a double buffer needs, the extra slots let the host link keep
        streaming the next pass's first layers for the whole draft-tree build
        (8 x 1.7 GB covers ~250 ms of PCIe time at 55 GB/s).
        tp: a communicator (tp.NcclComm / tp.ThreadComm) -> this model is rank
        tp.rank's tensor-parallel shard of the target (tp.py); the partial sums
        of the o / down projections are all-reduced in bf16 (reduce_bf16) or fp32.
        tp_fused: instead of a separate all-reduce, the projection's GEMM epilogue
        writes each feature slice of its bf16 partial into the owner rank's inbox
        over peer memory (sx_gemm_bf16_rs) and the owner reduces and broadcasts
        the slice (sx_tp_reduce_bcast). None = fused when the communicator
        provides peer memory, else the NCCL all-reduce.
        tp_argmax (KV1, t = 0 SpecExec only): the tree pass returns one int64
        argmax key per row (sx_rows_argmax_packed on this rank's vocab slice, an
        int64 MAX all-reduce over the ranks) instead of all-gathering the logit
        slices into [N, V]; the acceptance walk needs nothing else at t = 0, and
        a t > 0 walk or a full-row request raises."""
        if isinstance(cfg, str):
            cfg = PRESETS[cfg]
        if cfg.head_dim != 128:
            raise ValueError("head_dim must be 128")
        if dtype not in ("bf16", "fp32"):
            raise ValueError(f"dtype must be 'bf16' or 'fp32', got {dtype!r}")
        # fp32 target mode (csrc/fp32_path.cu): fp32 weights / activations / KV, FFMA GEMMs
        self.fp32 = dtype == "fp32"
        if self.fp32 and (offload or (tp is not None and tp.world > 1)):
            raise ValueError("the fp32 target mode runs resident on one GPU (no offload / tensor parallelism)")
        if not torch.cuda.is_available():
            raise RuntimeError("LlamaModel needs a CUDA device; there is no CPU fallback")
        _lib.load()
        self.cfg = cfg
        self.vocab_size = cfg.vocab
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.seed = seed
        self.tp = tp if (tp is not None and tp.world > 1) else None
        self.tp_argmax = bool(tp_argmax and self.tp is not None)
        self.shard = TPShard(tp.rank, tp.world) if self.tp is not None else None
        if self.shard is not None:
            self.shard.check(cfg)
        self.reduce_bf16 = bool(reduce_bf16 and self.tp is not None)
        self.H = cfg.heads // (self.tp.world if self.tp else 1)  # local query / KV heads
        self.KVH = cfg.kv_heads // (self.tp.world if self.tp else 1)
        wdt = torch.float32 if self.fp32 else torch.bfloat16
        self.dtype = dtype
        self.w = LlamaWeights(cfg, seed, self.device, std, lm_scale, offload=offload, shard=self.shard, init=init,
                              dtype=wdt)
        self.streamer = LayerStreamer(self.w, self.device, nbuf=max(2, min(offload_buffers, cfg.layers))) if offload else None
        self.slots = max_ctx
        self.kc = torch.zeros((cfg.layers, self.KVH, max_ctx, cfg.head_dim), dtype=wdt, device=self.device)
        self.vc = torch.zeros_like(self.kc)
        self.layer_stride = self.KVH * max_ctx * cfg.head_dim
        self.cos, self.sin = _rope_tables(cfg, max_ctx + 64, self.device)
        self.max_tokens = max_tokens
        self.buf = _Buffers(cfg, max_tokens, self.device, self.shard, self.reduce_bf16, act_dtype=wdt)
        self.tp_fused = False
        if self.tp is not None and tp_fused is not False:
            W = self.tp.world
            try:
                if cfg.d % (W * 128):
                    raise ValueError(f"fused TP reduce-scatter needs d={cfg.d} divisible by 128 x {W}")
                self.inbox, self.inbox_peers = self.tp.symm_buffer(W * max_tokens * (cfg.d // W), torch.bfloat16)
                ydt = torch.bfloat16 if self.reduce_bf16 else torch.float32
                ybuf, self.y_peers = self.tp.symm_buffer(max_tokens * cfg.d, ydt)
                self.buf.y = ybuf.view(max_tokens, cfg.d)  # peers write the reduced slices into it
                self.tp_fused = True
            except Exception as e:  # noqa: BLE001
                if tp_fused:
                    raise
                import sys

                print(f"[llama] fused TP reduce-scatter unavailable ({e}); using the NCCL all-reduce", file=sys.stderr)
        self.synthetic = synthetic
        if synthetic is not None:
            g = torch.Generator(device=self.device)
            g.manual_seed(synthetic.seed)
            self.bias_u = torch.empty((cfg.vocab, synthetic.rank), dtype=torch.bfloat16, device=self.device).normal_(
                0.0, 1.0, generator=g)
            self.bias_w = (torch.empty((cfg.vocab, synthetic.rank), dtype=torch.bfloat16, device=self.device)
                           .normal_(0.0, 1.0, generator=g) * (synthetic.scale / math.sqrt(synthetic.rank))).bfloat16()
            if self.fp32:  # the same (bf16-valued) table, held in fp32 for the FFMA GEMM
                self.bias_u, self.bias_w = self.bias_u.float(), self.bias_w.float()
            self.bias_in = torch.empty((max_tokens, synthetic.rank), dtype=wdt, device=self.device)
        self.committed: list[int] = []  # tokens whose KV is in slots [0, len)
        self.record: list[dict] | None = None  # test hook: per build, prefix -> fp32 logits row
        self.use_graphs = True  # draft rounds and one-token chains as CUDA graphs
        self.fuse_rope = True  # RoPE + KV-cache scatter fused into the QKV GEMM epilogue
        self._one_args = torch.zeros(4, dtype=torch.int32, device=self.device)
        self._g1 = None
        self._g1_out = None
        self._g1_warm = False
        LlamaModel._serial += 1
        self._uid = LlamaModel._serial
        self.stats = {"forward_tokens": 0, "forwards": 0}

    def draft_view(self) -> "LlamaModel":
        """The same network (weights, buffers, communicator shared) with its own
        KV cache and prefix state, for the draft role when a caller passes one
        model as both draft and target (the reference CLI's default,
        pkg/src/speckit/harness/cli.py:91): the roles keep different committed
        prefixes and tree slots, so they cannot share one cache. Created once."""
        v = getattr(self, "_draft_view_model", None)
        if v is None:
            v = object.__new__(type(self))
            v.__dict__.update(self.__dict__)
            v.kc = torch.zeros_like(self.kc)
            v.vc = torch.zeros_like(self.vc)
            v.committed = []
            v.record = None
            v._one_args = torch.zeros(4, dtype=torch.int32, device=self.device)
            v._g1, v._g1_out, v._g1_warm = None, None, False
            LlamaModel._serial += 1
            v._uid = LlamaModel._serial
            v.stats = {"forward_tokens": 0, "forwards": 0}
            v._draft_view_model = v
            self._draft_view_model = v
        return v

    # ------------------------------------------------------------------ forward
    def forward(self, n: int, tokens: torch.Tensor, pos: torch.Tensor | None, pos_base: int, slot: torch.Tensor | None,
                slot_base: int, dense_len: torch.Tensor | None, dense_const: int, anc: torch.Tensor | None,
                anc_base: int, anc_len: torch.Tensor | None, A: int, logits_from: int | None,
                argmax_only: bool = False) -> torch.Tensor | None:
        """Run n tokens through the network; write their K/V into the cache.

        Token t sits at position pos_base + pos[t] (pos None: t) and KV slot
        slot_base + slot[t]; it attends slots [0, dense_len[t]) and the anc
        list. Returns fp32 logits of rows [logits_from, n) (None: no LM head)."""
        cfg, b, w = self.cfg, self.buf, self.w
        if n > b.n:
            raise ValueError(f"forward of {n} tokens exceeds max_tokens={b.n}")
        if self.fp32:
            return self._forward_f32(n, tokens, pos, pos_base, slot, slot_base, dense_len, dense_const, anc, anc_base,
                                     anc_len, A, logits_from)
        st = _lib.stream_ptr()
        x, h = b.x[:n], b.h[:n]
        _lib.call("sx_embed", _lib.ptr(w.emb), _lib.ptr(tokens), n, cfg.d, _lib.ptr(x), st)
        p = _lib.ptr
        y = b.y[:n]
        tp, ybf = self.tp, int(self.reduce_bf16)
        epi_y = K.EPI_BF16 if ybf else K.EPI_F32
        H, KVH = self.H, self.KVH
        attn_ws_bytes = int(_lib.load().sx_tree_attention_ws_bytes(n, H, KVH))  # key-split partials (small grids)
        attn_ws = K.scratch(attn_ws_bytes, self.device, "attn", zero=True) if attn_ws_bytes > 0 else None
        for li in range(cfg.layers):
            L = self.streamer.acquire(li) if self.streamer is not None else w.layers[li]
            kc, vc = self.kc[li], self.vc[li]
            if li == 0:
                _lib.call("sx_rmsnorm", p(x), p(L["n1"]), n, cfg.d, cfg.eps, p(h), st)
            else:  # residual add of the previous layer's down projection, fused into this norm
                _lib.call("sx_add_rmsnorm", p(x), p(y), ybf, p(L["n1"]), n, cfg.d, cfg.eps, p(h), st)
            if self.fuse_rope:  # RoPE + KV scatter in the QKV GEMM epilogue
                K.gemm_qkv_rope(h, L["wqkv"], H, KVH, pos, pos_base, slot, slot_base, self.cos, self.sin, b.q[:n],
                                kc, vc, self.slots)
            else:
                K.gemm(h, L["wqkv"], out=b.qkv[:n])
                _lib.call("sx_rope_kv", p(b.qkv), p(pos), pos_base, p(slot), slot_base, n, H, KVH,
                          p(self.cos), p(self.sin), p(b.q), p(kc), p(vc), self.slots, st)
            _lib.call("sx_tree_attention_ws", p(b.q), p(kc), p(vc), self.slots, p(dense_len), dense_const, p(anc),
                      anc_base, p(anc_len), A, p(b.att), n, H, KVH, p(attn_ws), attn_ws_bytes, st)
            if self.tp_fused:
                self._fused_reduce(b.att[:n], L["wo"], n)
            else:
                K.gemm(b.att[:n], L["wo"], out=y, epi=epi_y)
                if tp is not None:
                    tp.all_reduce_(y)
            _lib.call("sx_add_rmsnorm", p(x), p(y), ybf, p(L["n2"]), n, cfg.d, cfg.eps, p(h), st)
            K.gemm(h, L["wgu"], out=b.act[:n], epi=K.EPI_SWIGLU_IL)
            if self.tp_fused:
                self._fused_reduce(b.act[:n], L["wd"], n)
            else:
                K.gemm(b.act[:n], L["wd"], out=y, epi=epi_y)
                if tp is not None:
                    tp.all_reduce_(y)
            if self.streamer is not None:
                self.streamer.release(li)
        self.stats["forward_tokens"] += n
        self.stats["forwards"] += 1
        if logits_from is None:
            return None
        m = n - logits_from
        hh = b.h[logits_from:n]
        _lib.call("sx_add_rmsnorm", p(x[logits_from:]), p(y[logits_from:]), ybf, p(w.nf), m, cfg.d, cfg.eps, p(hh), st)
        logits = b.logits[:m]
        if tp is not None and argmax_only:  # KV1: packed argmax keys of this slice, MAX-reduced over the ranks
            ll = b.logits_l[:m]
            K.gemm(hh, w.lm, out=ll, epi=K.EPI_F32)
            v0, v1 = self.shard.vocab(cfg)
            if self.synthetic is not None:
                bi = self.bias_in[:m]
                torch.index_select(self.bias_u, 0, tokens[logits_from:n].long(), out=bi)
                K.gemm(bi, self.bias_w[v0:v1], out=ll, epi=K.EPI_ADD_F32)
            keys = b.argmax_keys[:m]
            K.rows_argmax_packed(ll, v0, keys)
            tp.max_reduce_(keys)
            return keys
        if tp is None:
            K.gemm(hh, w.lm, out=logits, epi=K.EPI_F32)
        else:  # vocab-parallel LM head: local slice, all-gather, interleave the slices into [m, V]
            ll = b.logits_l[:m]
            K.gemm(hh, w.lm, out=ll, epi=K.EPI_F32)
            gather_vocab(tp, ll, logits, b.logits_g)
        if self.synthetic is not None:
            bi = self.bias_in[:m]
            torch.index_select(self.bias_u, 0, tokens[logits_from:n].long(), out=bi)
            K.gemm(bi, self.bias_w, out=logits, epi=K.EPI_ADD_F32)
        return logits

    def _forward_f32(self, n, tokens, pos, pos_base, slot, slot_base, dense_len, dense_const, anc, anc_base, anc_len, A,
                     logits_from):
        """The fp32 target mode: the same sequence of operations as `forward`,
        every tensor fp32, FFMA GEMMs and the fp32 attention (csrc/fp32_path.cu)."""
        cfg, b, w = self.cfg, self.buf, self.w
        st, p = _lib.stream_ptr(), _lib.ptr
        x, h, y = b.x[:n], b.h[:n], b.y[:n]
        H, KVH = self.H, self.KVH
        _lib.call("sx_embed_f32", p(w.emb), p(tokens), n, cfg.d, p(x), st)

        def gemm(xin, wt, out, epi):
            _lib.call("sx_gemm_f32", p(wt), p(xin), p(out), xin.shape[0], wt.shape[0], wt.shape[1], out.stride(0), epi,
                      st)

        for li in range(cfg.layers):
            L = w.layers[li]
            kc, vc = self.kc[li], self.vc[li]
            _lib.call("sx_add_rmsnorm_f32", p(x), p(y) if li > 0 else None, p(L["n1"]), n, cfg.d, cfg.eps, p(h), st)
            gemm(h, L["wqkv"], b.qkv[:n], K.EPI_F32)
            _lib.call("sx_rope_kv_f32", p(b.qkv), p(pos), pos_base, p(slot), slot_base, n, H, KVH, p(self.cos),
                      p(self.sin), p(b.q), p(kc), p(vc), self.slots, st)
            _lib.call("sx_tree_attention_f32", p(b.q), p(kc), p(vc), self.slots, p(dense_len), dense_const, p(anc),
                      anc_base, p(anc_len), A, p(b.att), n, H, KVH, st)
            gemm(b.att[:n], L["wo"], y, K.EPI_F32)
            _lib.call("sx_add_rmsnorm_f32", p(x), p(y), p(L["n2"]), n, cfg.d, cfg.eps, p(h), st)
            gemm(h, L["wgu"], b.act[:n], K.EPI_SWIGLU_IL)
            gemm(b.act[:n], L["wd"], y, K.EPI_F32)
        self.stats["forward_tokens"] += n
        self.stats["forwards"] += 1
        if logits_from is None:
            return None
        m = n - logits_from
        hh = b.h[logits_from:n]
        _lib.call("sx_add_rmsnorm_f32", p(x[logits_from:]), p(y[logits_from:]), p(w.nf), m, cfg.d, cfg.eps, p(hh), st)
        logits = b.logits[:m]
        gemm(hh, w.lm, logits, K.EPI_F32)
        if self.synthetic is not None:
            bi = self.bias_in[:m]
            torch.index_select(self.bias_u, 0, tokens[logits_from:n].long(), out=bi)
            gemm(bi, self.bias_w, logits, K.EPI_ADD_F32)
        return logits

    def _fused_reduce(self, xin: torch.Tensor, w: torch.Tensor, n: int) -> None:
        """y[:n] = sum over ranks of xin @ w^T: GEMM + reduce-scatter over peer
        memory, barrier, owner reduce + broadcast, barrier."""
        tp = self.tp
        K.gemm_rs(xin, w, self.inbox_peers, tp.rank, tp.world)
        tp.barrier_device()
        _lib.call("sx_tp_reduce_bcast", _lib.ptr(self.inbox), tp.rank, tp.world, n, self.cfg.d, _lib.ptr(self.y_peers),
                  int(self.reduce_bf16), _lib.stream_ptr())
        tp.barrier_device()

    # ---------------------------------------------------------- prefix cache
    def _sync(self, prefix: tuple[int, ...]) -> tuple[int, list[int]]:
        """Keep the longest committed prefix of `prefix[:-1]`; return (c, pending)
        where pending = prefix[c:] (always non-empty; its last token is the root)."""
        c = 0
        lim = min(len(self.committed), len(prefix) - 1)
        while c < lim and self.committed[c] == prefix[c]:
            c += 1
        del self.committed[c:]
        return c, list(prefix[c:])

    def _chain_one(self, c: int, token: int) -> torch.Tensor:
        """One token at slot/position c with logits -- the draft's first round of
        every tree (the root) and each step of sequential decoding -- replayed as
        a CUDA graph (per-token scalars live in a device array, so one capture
        serves every c). The first call runs eagerly to settle kernel attributes
        and tensor maps, the second captures."""
        if c + 1 > self.slots:
            raise RuntimeError(f"KV cache full ({self.slots} slots)")
        a = self._one_args
        a.copy_(torch.tensor([token, c, c, c + 1], dtype=torch.int32), non_blocking=True)
        K.IO["h2d"] += 16
        tok, pos, slot, dl = a[0:1], a[1:2], a[2:3], a[3:4]
        if self._g1 is None and self._g1_warm:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            n0 = _lib.load().sx_launch_count()
            with torch.cuda.graph(g):
                self._g1_out = self.forward(1, tok, pos, 0, slot, 0, dl, 0, None, 0, None, 0, 0)
            self._g1_kernels = _lib.load().sx_launch_count() - n0
            self._g1 = g
        if self._g1 is not None:
            self._g1.replay()
            K.GRAPH_KERNELS[0] += self._g1_kernels
            out = self._g1_out
            self.stats["forward_tokens"] += 1
            self.stats["forwards"] += 1
        else:
            out = self.forward(1, tok, pos, 0, slot, 0, dl, 0, None, 0, None, 0, 0)
            self._g1_warm = True
        self.committed.append(int(token))
        return out

    def _chain(self, c: int, toks: Sequence[int], want_logits: bool) -> torch.Tensor | None:
        """Causal chain of tokens at slots/positions c.. (prefill, catch-up)."""
        if len(toks) == 1 and want_logits and self.use_graphs and self.streamer is None and self.tp is None:
            return self._chain_one(c, toks[0])
        out = None
        i = 0
        step = self.buf.n
        while i < len(toks):
            chunk = toks[i : i + step]
            n = len(chunk)
            base = c + i
            if base + n > self.slots:
                raise RuntimeError(f"KV cache full ({self.slots} slots)")
            tok = self.buf.tok[:n]
            tok.copy_(torch.tensor(chunk, dtype=torch.int32), non_blocking=True)
            K.IO["h2d"] += 8 * n
            dl = self.buf.pos[:n]
            dl.copy_(torch.arange(base + 1, base + n + 1, dtype=torch.int32), non_blocking=True)
            last = i + n >= len(toks)
            out = self.forward(n, tok, None, base, None, base, dl, 0, None, 0, None, 0,
                               (n - 1) if (want_logits and last) else None)
            i += n
        self.committed.extend(int(t) for t in toks)
        return out

    def prefix_rows(self, prefix) -> torch.Tensor:
        """fp32 logits [1, V] of the next token after `prefix` (commits the prefix)."""
        prefix = _check_prefix(prefix, self.vocab_size)
        if not prefix:
            raise ValueError("empty prefix")
        c, pending = self._sync(prefix)
        return self._chain(c, pending, True)

    def next_distributions(self, prefixes) -> np.ndarray:
        rows = [K.softmax_rows(self.prefix_rows(p))[0].cpu().numpy() for p in prefixes]
        if not rows:
            return np.empty((0, self.vocab_size))
        return np.stack(rows)

    # -------------------------------------------------- device-model protocol
    def tree_session(self, prefix, params: BuilderParams) -> "_LlamaDraftSession":
        _check_prefix(prefix, self.vocab_size)
        return _LlamaDraftSession(self, tuple(prefix), params)

    def stochastic_session(self, prefix, max_nodes: int, max_depth: int) -> "_LlamaStochastic":
        _check_prefix(prefix, self.vocab_size)
        return _LlamaStochastic(self, tuple(prefix), max_nodes, max_depth)

    def tree_rows(self, tree) -> torch.Tensor:
        """ONE target pass over the anchor + every tree node: fp32 logits [n+1, V]."""
        prefix = tree.prefix
        c, pending = self._sync(prefix)
        if len(pending) > 1:
            self._chain(c, pending[:-1], False)
            c += len(pending) - 1
        n = len(tree) + 1
        if c + n > self.slots:
            raise RuntimeError(f"KV cache full: need {c + n} slots, have {self.slots}")
        ws = tree.workspace
        if ws is not None:
            anc, anc_len, depth, tok = ws.final_tables(n)
            A = ws.D + 1
        else:  # host-built tree (SpecInfer): same tables, uploaded
            tabs = tree_tables(tree)
            anc, anc_len, depth, tok = (torch.from_numpy(a).to(self.device, non_blocking=True) for a in tabs)
            A = tabs[0].shape[1]
            K.IO["h2d"] += sum(a.nbytes for a in tabs)
        if self.tp_argmax and self.record is not None:
            raise RuntimeError("tp_argmax keeps no logit rows; the replay record needs them")
        logits = self.forward(n, tok, depth, c, None, c, None, c, anc, c, anc_len, A, 0, argmax_only=self.tp_argmax)
        self.committed.append(prefix[-1])  # the root's KV is at slot c = its position
        tree.target_base = c
        if self.record is not None:
            rows = logits.cpu().numpy()
            rec = {prefix: rows[0].copy()}
            for node in tree.nodes:
                rec[tree.full_prefix(node.node_id)] = rows[node.node_id + 1].copy()
            self.record.append(rec)
        return logits

    def commit_walk(self, cache, res) -> None:
        """Move the accepted path's KV into the committed region after a walk."""
        tree = cache.tree
        if getattr(cache, "target", None) is self and hasattr(tree, "target_base"):
            c = tree.target_base
            rows = [r for r in res.path_rows]
            if rows:
                src = torch.tensor([c + r for r in rows], dtype=torch.int32).to(self.device, non_blocking=True)
                dst = torch.tensor([c + 1 + i for i in range(len(rows))], dtype=torch.int32).to(self.device,
                                                                                                 non_blocking=True)
                _lib.call("sx_kv_compact_f32" if self.fp32 else "sx_kv_compact", _lib.ptr(self.kc), _lib.ptr(self.vc),
                          self.cfg.layers, self.layer_stride, self.slots, self.KVH, _lib.ptr(src), _lib.ptr(dst),
                          len(rows), _lib.stream_ptr())
                K.IO["h2d"] += 8 * len(rows)
            self.committed.extend(tree.nodes[r - 1].token for r in rows)
        elif getattr(tree, "draft_model", None) is self:
            c = tree.draft_root_slot
            if hasattr(tree, "host_slot"):  # host-built (SpecInfer) tree
                slots = tree.host_slot
            else:  # GPU-built tree: slots staged with the nodes
                tree.nodes  # noqa: B018
                slots = tree.host_slot_staged
            src, toks = [], []
            for r in res.path_rows:
                s = slots[r - 1]
                if s < 0:
                    break
                src.append(s)
                toks.append(tree.nodes[r - 1].token)
            if src:
                s_t = torch.tensor(src, dtype=torch.int32).to(self.device, non_blocking=True)
                d_t = torch.tensor([c + 1 + i for i in range(len(src))], dtype=torch.int32).to(self.device,
                                                                                                non_blocking=True)
                _lib.call("sx_kv_compact_f32" if self.fp32 else "sx_kv_compact", _lib.ptr(self.kc), _lib.ptr(self.vc),
                          self.cfg.layers, self.layer_stride, self.slots, self.KVH, _lib.ptr(s_t), _lib.ptr(d_t),
                          len(src), _lib.stream_ptr())
                K.IO["h2d"] += 8 * len(src)
            self.committed.extend(toks)


class _LlamaDraftSession:
    """Feeds the GPU tree builder: round 1 = catch-up chain + root, later rounds
    = the batch nodes with their ancestor KV slots (tree.py:282-296)."""

    def __init__(self, model: LlamaModel, prefix: tuple[int, ...], params: BuilderParams):
        self.m = model
        self.prefix = prefix
        self.ws = _WS.get(params.budget, params.batch_size, model.vocab_size, params.max_depth)
        c, pending = model._sync(prefix)
        self.c, self.pending = c, pending
        self.root_slot = c + len(pending) - 1
        self.ws.begin(root_slot=self.root_slot, pad_slot=model.slots - 1)
        self.first = True
        self.batch_n = 1
        self.rec = None
        if model.record is not None:  # replay-oracle hook: prefix -> fp32 logits of this build
            self.rec = {}
            self.slot_path = {self.root_slot: ()}
            model.record.append(self.rec)

    def batch_rows(self) -> torch.Tensor:
        m = self.m
        if self.first:
            self.first = False
            out = m._chain(self.c, self.pending, True)
            if self.rec is not None:
                self.rec[self.prefix] = out[0].cpu().numpy().copy()
            return out
        ws, n = self.ws, self.batch_n
        out = m.forward(n, ws.batch_tokens()[:n], ws.batch_pos()[:n], 0, ws.batch_slots()[:n], 0, None, self.root_slot,
                        ws.batch_anc()[:n], 0, ws.batch_anc_len()[:n], ws.D + 1, 0)
        if self.rec is not None:
            anc, alen = ws.batch_anc()[:n].cpu().tolist(), ws.batch_anc_len()[:n].cpu().tolist()
            toks, slots = ws.batch_tokens()[:n].cpu().tolist(), ws.batch_slots()[:n].cpu().tolist()
            rows = out.cpu().numpy()
            for b in range(n):
                path = self.slot_path[anc[b][alen[b] - 2]] + (toks[b],)
                self.slot_path[slots[b]] = path
                self.rec[self.prefix + path] = rows[b].copy()
        return out

    # -- fused round: fixed-shape draft forward over all B batch rows (rows past
    # batch_n are padding that writes only the scratch slot) + scoring + update,
    # replayed as one CUDA graph per (model, workspace, scoring mode).
    def _bucket(self) -> int:
        """Rows the fixed-shape round runs: the smallest power of two (>= 32)
        covering the current batch, capped at B -- deep trees expand a few
        frontier nodes per round; padding every round to B wasted the draft."""
        B, n = self.ws.B, 32
        while n < self.batch_n and n < B:
            n *= 2
        return min(n, B)

    def run_round(self, mode: int, temp: float, top_p: float) -> dict:
        m, ws = self.m, self.ws
        if self.first or not m.use_graphs or ws.B > m.buf.n:
            rows = self.batch_rows()
            return ws.round(rows, mode, temp, top_p)
        snap = self._snapshot() if self.rec is not None else None
        if not hasattr(ws, "_graphs"):
            ws._graphs = {}
        n = self._bucket()
        key = (m._uid, mode, temp, top_p, n)
        g = ws._graphs.get(key)
        if g is None:
            if key not in getattr(ws, "_graph_warm", set()):
                # one eager fixed-shape round first (sets kernel attributes, tensor maps, scratch)
                ws._graph_warm = getattr(ws, "_graph_warm", set()) | {key}
                self._fixed_forward(n)
                ws.launch_round(m.buf.logits[:n], mode, temp, top_p)
                ctl = ws.read_ctl()
                self._record(snap)
                return ctl
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            n0 = _lib.load().sx_launch_count()
            with torch.cuda.graph(g):
                self._fixed_forward(n)
                ws.launch_round(m.buf.logits[:n], mode, temp, top_p)
            g.sx_kernels = _lib.load().sx_launch_count() - n0
            ws._graphs[key] = g
        ws.last_round = (m.buf.logits[:n], mode, temp, top_p)  # rows of a sliced re-run on survivor overflow
        g.replay()
        K.GRAPH_KERNELS[0] += g.sx_kernels
        ctl = ws.read_ctl()
        self._record(snap)
        return ctl

    def _snapshot(self):
        ws, n = self.ws, self.batch_n
        return (ws.batch_anc()[:n].cpu().tolist(), ws.batch_anc_len()[:n].cpu().tolist(),
                ws.batch_tokens()[:n].cpu().tolist(), ws.batch_slots()[:n].cpu().tolist())

    def _record(self, snap) -> None:
        if snap is None:
            return
        anc, alen, toks, slots = snap
        rows = self.m.buf.logits[: len(toks)].cpu().numpy()
        for b in range(len(toks)):
            path = self.slot_path[anc[b][alen[b] - 2]] + (toks[b],)
            self.slot_path[slots[b]] = path
            self.rec[self.prefix + path] = rows[b].copy()

    def _fixed_forward(self, n: int) -> None:
        ws = self.ws
        self.m.forward(n, ws.batch_tokens()[:n], ws.batch_pos()[:n], 0, ws.batch_slots()[:n], 0,
                       ws.batch_dense()[:n], 0, ws.batch_anc()[:n], 0, ws.batch_anc_len()[:n], ws.D + 1, 0)

    def advance(self, ctl) -> None:
        self.batch_n = ctl["batch_n"]
        if ctl["slot_next"] >= self.m.slots:
            raise RuntimeError(f"draft KV slots exhausted ({ctl['slot_next']} >= {self.m.slots}); raise max_ctx")
        if self.batch_n > self.m.buf.n:
            raise RuntimeError("draft batch exceeds max_tokens")

    def finish(self, tree) -> None:
        tree.draft_model = self.m
        tree.draft_root_slot = self.root_slot  # node KV slots arrive with the staged tree (host_slot_staged)


class _LlamaStochastic:
    """Level-by-level draft rows for SpecInfer's stochastic builder
    (tree.py:383-425): the root row by the usual catch-up chain, then each level
    in one forward where node i sits at KV slot root+1+i and attends the
    committed prefix, the root and its ancestors (host-built ancestor lists)."""

    def __init__(self, model: LlamaModel, prefix: tuple[int, ...], max_nodes: int, max_depth: int):
        self.m = model
        self.prefix = prefix
        c, pending = model._sync(prefix)
        self.c, self.pending = c, pending
        self.root_slot = c + len(pending) - 1
        if self.root_slot + 1 + max_nodes > model.slots:
            raise RuntimeError(f"draft KV slots exhausted ({self.root_slot + 1 + max_nodes} > {model.slots})")
        self.A = max_depth + 1
        self.expanded: set[int] = set()
        self.rec = None
        if model.record is not None:  # replay-oracle hook: prefix -> fp32 logits of this build
            self.rec = {}
            model.record.append(self.rec)

    def level_rows(self, tree, level: list[int]) -> torch.Tensor:
        out = self._level_rows(tree, level)
        if self.rec is not None:
            rows = out.cpu().numpy()
            for j, nid in enumerate(level):
                self.rec[tree.full_prefix(nid)] = rows[j].copy()
        return out

    def _level_rows(self, tree, level: list[int]) -> torch.Tensor:
        m = self.m
        if level == [-1]:
            return m._chain(self.c, self.pending, True)
        n = len(level)
        if n > m.buf.n:
            raise RuntimeError(f"SpecInfer level of {n} nodes exceeds max_tokens={m.buf.n}")
        anc = np.zeros((n, self.A), dtype=np.int32)
        alen = np.zeros(n, dtype=np.int32)
        depth = np.zeros(n, dtype=np.int32)
        slot = np.zeros(n, dtype=np.int32)
        tok = np.zeros(n, dtype=np.int32)
        rs = self.root_slot
        for j, nid in enumerate(level):
            chain = []
            x = nid
            while x != -1:
                chain.append(rs + 1 + x)
                x = tree.nodes[x].parent
            chain.append(rs)
            chain.reverse()
            anc[j, : len(chain)] = chain
            alen[j] = len(chain)
            depth[j] = tree.nodes[nid].depth
            slot[j] = 1 + nid
            tok[j] = tree.nodes[nid].token
        dev = m.device
        t_anc, t_alen, t_depth, t_slot, t_tok = (torch.from_numpy(a).to(dev, non_blocking=True)
                                                  for a in (anc, alen, depth, slot, tok))
        K.IO["h2d"] += int(anc.nbytes + 4 * 4 * n)
        self.expanded.update(level)
        return m.forward(n, t_tok, t_depth, rs, t_slot, rs, None, rs, t_anc, 0, t_alen, self.A, 0)

    def finish(self, tree) -> None:
        """KV bookkeeping for commit_walk: nodes whose KV the draft computed."""
        tree.draft_model = self.m
        tree.draft_root_slot = self.root_slot
        tree.host_slot = [self.root_slot + 1 + i if i in self.expanded else -1 for i in range(len(tree.nodes))]
