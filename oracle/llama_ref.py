"""fp32 CPU reference forward of the Llama architecture. TEST INFRASTRUCTURE.

The floating-point reference for the target / draft logits of the B200 path
(north_star tolerance: 2e-2 abs in bf16). Plain PyTorch on the CPU, fp32, full
causal attention over an explicit token prefix -- i.e. exactly what the
reference's stateless `LanguageModel.next_distributions(prefixes)`
(pkg/src/speckit/models.py:47-52) means for a Llama-shaped model: no KV cache,
no tree mask, no kernels. HF Llama conventions: RMSNorm, rotate-half RoPE
(theta from the config), GQA by repeating KV heads, SwiGLU MLP, untied LM head.
"""

from __future__ import annotations

import numpy as np
import torch


def rope(x: torch.Tensor, pos: torch.Tensor, theta: float) -> torch.Tensor:
    hd = x.shape[-1]
    inv_freq = 1.0 / (theta ** (torch.arange(0, hd, 2, dtype=torch.int64).float() / hd))
    freqs = torch.outer(pos.float(), inv_freq)
    cos, sin = freqs.cos()[:, None, :], freqs.sin()[:, None, :]
    x0, x1 = x[..., : hd // 2], x[..., hd // 2 :]
    return torch.cat([x0 * cos - x1 * sin, x1 * cos + x0 * sin], dim=-1)


def rmsnorm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


@torch.no_grad()
def forward_logits(cfg, W: dict, tokens: list[int], bias=None, layers: int | None = None,
                   policy: str = "fp32") -> torch.Tensor:
    """fp32 logits [len(tokens), V] for every position of a causal prefix."""
    n = len(tokens)
    mask = torch.full((n, n), float("-inf")).triu(1)
    return forward_masked(cfg, W, tokens, torch.arange(n), mask, bias, layers, policy)


@torch.no_grad()
def forward_tree_logits(cfg, W: dict, prompt: list[int], paths: list[tuple[int, ...]], bias=None,
                        layers: int | None = None, policy: str = "fp32") -> torch.Tensor:
    """fp32 logits [1 + len(paths), V]: row 0 = the next token after `prompt`,
    row 1 + i = the next token after prompt + paths[i] -- what the reference's
    `precompute` asks of the target (pkg/src/speckit/engine.py:73-89): one row
    per tree prefix. `paths` must be prefix-closed (every non-empty path's
    parent path is listed, or is the empty root path) and parents must come
    first. One forward over prompt + tree tokens with the flattened ancestor
    mask of pkg/src/speckit/tree.py:208-219 (node i sees the prompt, its
    ancestors and itself) at position len(prompt) - 1 + depth; each row is
    mathematically the causal forward of its full prefix (checked by
    tests/test_llama_ref_cpu.py)."""
    P, n = len(prompt), len(paths)
    index = {(): P - 1}  # path -> sequence row (the root = the prompt's last token)
    toks = list(prompt)
    pos = list(range(P))
    parent_row = []
    for i, path in enumerate(paths):
        if len(path) == 0 or path[:-1] not in index:
            raise ValueError(f"paths must be non-empty and prefix-closed, parents first (path {i})")
        index[tuple(path)] = P + i
        toks.append(int(path[-1]))
        pos.append(P - 1 + len(path))
        parent_row.append(index[path[:-1]])
    T = P + n
    allow = torch.zeros((T, T), dtype=torch.bool)
    allow[:P, :P] = torch.ones((P, P), dtype=torch.bool).tril()
    for i in range(n):  # parents first: copy the parent's visibility, add self
        r = P + i
        allow[r] = allow[parent_row[i]]
        allow[r, r] = True
    mask = torch.zeros((T, T)).masked_fill(~allow, float("-inf"))
    logits = forward_masked(cfg, W, toks, torch.tensor(pos), mask, bias, layers, policy)
    return torch.cat([logits[P - 1 : P], logits[P:]], dim=0)


@torch.no_grad()
def forward_masked(cfg, W: dict, tokens: list[int], pos: torch.Tensor, mask: torch.Tensor, bias=None,
                   layers: int | None = None, policy: str = "fp32") -> torch.Tensor:
    """fp32 logits of every row of `tokens` at positions `pos` under an additive
    attention mask [n, n] (0 = visible, -inf = masked).

    policy="fp32": every activation in fp32 (the reference's meaning of the
    model). policy="bf16": the same arithmetic with activations rounded to bf16
    exactly where the B200 bf16 path stores them (the GEMM operands: normed
    inputs, RoPE'd q / k and v in the KV cache, the attention output, the SwiGLU
    product, the final normed row; residual stream and accumulators fp32) -- the
    precision policy the north_star's "2e-2 abs in bf16" is measured against."""
    if policy not in ("fp32", "bf16", "fp64"):
        raise ValueError(f"unknown precision policy {policy!r}")
    act = (lambda t: t.bfloat16().float()) if policy == "bf16" else (lambda t: t)
    wide = policy == "fp64"  # float64 arithmetic on the same weights: the exact-math yardstick of the fp32 mode
    up = (lambda t: t.double()) if wide else (lambda t: t)
    n = len(tokens)
    H, KVH, hd = cfg.heads, cfg.kv_heads, cfg.head_dim
    tok = torch.tensor(tokens, dtype=torch.long)
    x = up(W["emb"][tok].clone())
    if wide:
        mask = mask.double()
    for L in W["layers"][: layers if layers is not None else len(W["layers"])]:
        L = {k: up(v) for k, v in L.items()}
        h = act(rmsnorm(x, L["n1"], cfg.eps))
        qkv = h @ L["wqkv"].t()
        q = qkv[:, : H * hd].view(n, H, hd)
        k = qkv[:, H * hd : (H + KVH) * hd].view(n, KVH, hd)
        v = act(qkv[:, (H + KVH) * hd :].view(n, KVH, hd))
        q, k = act(rope(q, pos, cfg.rope_theta)), act(rope(k, pos, cfg.rope_theta))
        if wide:
            q, k = q.double(), k.double()
        g = H // KVH
        k = k.repeat_interleave(g, dim=1)
        v = v.repeat_interleave(g, dim=1)
        s = torch.einsum("qhd,khd->hqk", q, k) / hd**0.5 + mask
        att = act(torch.einsum("hqk,khd->qhd", s.softmax(-1), v).reshape(n, H * hd))
        x = x + att @ L["wo"].t()
        h = act(rmsnorm(x, L["n2"], cfg.eps))
        x = x + act(torch.nn.functional.silu(h @ L["wg"].t()) * (h @ L["wu"].t())) @ L["wd"].t()
    logits = act(rmsnorm(x, up(W["nf"]), cfg.eps)) @ up(W["lm"]).t()
    if bias is not None:
        u, w = bias
        logits = logits + up(u[tok]) @ up(w).t()
    return logits


@torch.no_grad()
def forward_logits_tp(cfg, W_local: dict, tokens: list[int], shard, all_reduce, all_gather) -> torch.Tensor:
    """The same forward on one rank of a tensor-parallel group: W_local holds this
    rank's slices (paper_2406_02532_b200/tp.py TPShard.shard), `all_reduce(t)`
    sums in place over the group, `all_gather(t) -> [world, *t.shape]`. Returns
    the full [len(tokens), V] logits on every rank. Checks the partition: it must
    reproduce forward_logits of the unsharded weights."""
    n = len(tokens)
    H, KVH, hd = cfg.heads // shard.world, cfg.kv_heads // shard.world, cfg.head_dim
    tok = torch.tensor(tokens, dtype=torch.long)
    x = W_local["emb"][tok].clone()
    pos = torch.arange(n)
    mask = torch.full((n, n), float("-inf")).triu(1)
    for L in W_local["layers"]:
        h = rmsnorm(x, L["n1"], cfg.eps)
        qkv = h @ L["wqkv"].t()
        q = qkv[:, : H * hd].view(n, H, hd)
        k = qkv[:, H * hd : (H + KVH) * hd].view(n, KVH, hd)
        v = qkv[:, (H + KVH) * hd :].view(n, KVH, hd)
        q, k = rope(q, pos, cfg.rope_theta), rope(k, pos, cfg.rope_theta)
        g = H // KVH
        k = k.repeat_interleave(g, dim=1)
        v = v.repeat_interleave(g, dim=1)
        s = torch.einsum("qhd,khd->hqk", q, k) / hd**0.5 + mask
        att = torch.einsum("hqk,khd->qhd", s.softmax(-1), v).reshape(n, H * hd)
        y = att @ L["wo"].t()
        all_reduce(y)
        x = x + y
        h = rmsnorm(x, L["n2"], cfg.eps)
        y = (torch.nn.functional.silu(h @ L["wg"].t()) * (h @ L["wu"].t())) @ L["wd"].t()
        all_reduce(y)
        x = x + y
    local = rmsnorm(x, W_local["nf"], cfg.eps) @ W_local["lm"].t()
    parts = all_gather(local)
    return torch.cat(list(parts), dim=1)


class CpuLlamaLM:
    """The reference plugin interface (pkg/src/speckit/models.py:32-63) over the
    fp32 CPU forward: `next_distributions(prefixes)` -> canonical float64 softmax
    rows (oracle.speckit_oracle.softmax_row, the rows the GPU computes from its
    fp32 logits). The TorchCpuLlama of SURVEY 8(c)/(d): the timed CPU reference
    path of bench.py's reference arm. A batch is evaluated as one tree-masked
    forward over the prefix closure of its prefixes below their common prefix
    (every row equals the stateless causal forward of its prefix)."""

    backend = "cpu-llama"

    def __init__(self, cfg, W: dict, policy: str = "fp32", threads: int | None = None):
        self.cfg, self.W, self.policy = cfg, W, policy
        self.vocab_size = cfg.vocab
        if threads:
            torch.set_num_threads(threads)

    def logits(self, prefixes) -> torch.Tensor:
        prefixes = [tuple(int(t) for t in p) for p in prefixes]
        if not prefixes:
            return torch.empty((0, self.vocab_size))
        if any(len(p) == 0 for p in prefixes):
            raise ValueError("empty prefix")
        c = min(len(p) for p in prefixes)
        first = prefixes[0]
        while c > 1 and any(p[:c] != first[:c] for p in prefixes):
            c -= 1
        anchor = list(first[:c])
        if any(p[:c] != first[:c] for p in prefixes):  # no shared token at all: one forward each
            return torch.stack([forward_logits(self.cfg, self.W, list(p), policy=self.policy)[-1] for p in prefixes])
        closure: dict[tuple[int, ...], None] = {}
        for p in prefixes:
            tail = p[c:]
            for j in range(1, len(tail) + 1):
                closure.setdefault(tail[:j], None)
        paths = sorted(closure, key=len)
        rows = forward_tree_logits(self.cfg, self.W, anchor, paths, policy=self.policy)
        at = {(): 0, **{q: i + 1 for i, q in enumerate(paths)}}
        return rows[[at[p[c:]] for p in prefixes]]

    def next_distributions(self, prefixes):
        from .speckit_oracle import softmax_row

        z = self.logits(prefixes).numpy().astype(np.float32)
        if z.shape[0] == 0:
            return np.empty((0, self.vocab_size))
        return np.stack([softmax_row(z[i]) for i in range(z.shape[0])])

    def next_distribution(self, prefix):
        return self.next_distributions([prefix])[0]
