"""In-situ vs isolated GEMM timing on 70B-shaped layers (2 layers, n = 1025):
per-shape CUDA-event times inside a real forward, then the o-projection
re-run in isolation on the forward's own buffers and on random inputs."""
import pathlib
import sys
from dataclasses import replace

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2406_02532_b200 import kernels as K  # noqa: E402
from paper_2406_02532_b200.llama import PRESETS, LlamaModel  # noqa: E402


def timeit(fn, n=10):
    fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3


cfg = replace(PRESETS["llama2-70b"], layers=2, name="70b-2L")
m = LlamaModel(cfg, seed=1, max_ctx=2048, max_tokens=1025)
toks = list(range(1, 1026))
m._chain(0, toks, True)
torch.cuda.synchronize()
m.committed.clear()
K.PROFILER = K.GemmProfiler()
m._chain(0, toks, True)
for r in K.PROFILER.by_shape(steps=1):
    print("in-situ", r)
K.PROFILER = None
b, L = m.buf, m.w.layers[0]
n = 1025
att, x = b.att[:n], b.x[:n]
print("att absmax", att.float().abs().max().item(), "x absmax", x.abs().max().item())
print("o isolated, model buffers : %.1f us" % timeit(lambda: K.gemm(att, L["wo"], out=x, epi=K.EPI_ADD_F32)))
ra = torch.randn_like(att.float()).bfloat16()
print("o isolated, random input  : %.1f us" % timeit(lambda: K.gemm(ra, L["wo"], out=x, epi=K.EPI_ADD_F32)))
xo = torch.zeros_like(x)
print("o isolated, fresh out     : %.1f us" % timeit(lambda: K.gemm(att, L["wo"], out=xo, epi=K.EPI_ADD_F32)))
wo = L["wo"].clone()
print("o isolated, cloned weight : %.1f us" % timeit(lambda: K.gemm(att, wo, out=x, epi=K.EPI_ADD_F32)))
print("o isolated, bf16 epilogue : %.1f us" % timeit(lambda: K.gemm(att, wo, out=b.q[:n], epi=K.EPI_BF16)))
print("qkv isolated             : %.1f us" % timeit(lambda: K.gemm(b.h[:n], L["wqkv"], out=b.qkv[:n])))

# what slows the o-projection down right after the attention kernel?
from paper_2406_02532_b200 import _lib  # noqa: E402

p, st, cfgm = _lib.ptr, _lib.stream_ptr(), m.cfg
pos = b.pos[:n]
pos.copy_(torch.arange(1, n + 1, dtype=torch.int32))
kc, vc = m.kc[0], m.vc[0]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
q2 = torch.empty_like(b.q[:n])


def attn(out=None):
    _lib.call("sx_tree_attention", p(b.q), p(kc), p(vc), m.slots, p(pos), 0, None, 0, None, 0,
              p(b.att if out is None else out), n, cfgm.heads, cfgm.kv_heads, st)


def t1(fn):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3


cases = {
    "o add (baseline)": (attn, lambda: K.gemm(att, L["wo"], out=x, epi=K.EPI_ADD_F32)),
    "o bf16 epilogue": (attn, lambda: K.gemm(att, L["wo"], out=b.q[:n], epi=K.EPI_BF16)),
    "qkv (reads h)": (attn, lambda: K.gemm(b.h[:n], L["wqkv"], out=b.qkv[:n])),
    "o reading a copy of att": (lambda: (attn(), q2.copy_(att)), lambda: K.gemm(q2, L["wo"], out=x, epi=K.EPI_ADD_F32)),
    "o after L2 flush": (lambda: (attn(), flush.fill_(1)), lambda: K.gemm(att, L["wo"], out=x, epi=K.EPI_ADD_F32)),
    "o after attention into q2": (lambda: attn(q2), lambda: K.gemm(att, L["wo"], out=x, epi=K.EPI_ADD_F32)),
    "o after rmsnorm only": (lambda: _lib.call("sx_rmsnorm", p(x), p(L["n1"]), n, cfgm.d, cfgm.eps, p(b.h), st),
                             lambda: K.gemm(att, L["wo"], out=x, epi=K.EPI_ADD_F32)),
}
for name, (pre, fn) in cases.items():
    res = []
    for _ in range(3):
        pre()
        torch.cuda.synchronize()
        res.append(t1(fn))
    print(f"{name:28s} " + " ".join(f"{r:7.1f}" for r in res) + " us")
