"""Where do GPU bf16 logits and the bf16-policy CPU oracle part ways? One-layer
truncation of a named architecture, one prefix: compares every intermediate the
forward leaves in its buffers (q, att, act, residual x, final normed h, logits)
with the oracle's bf16-policy restatement step by step. GPU tool (not a test)."""

import dataclasses
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import llama_ref  # noqa: E402
from paper_2406_02532_b200.llama import PRESETS, LlamaModel  # noqa: E402


def main(name="llama2-7b", n=1, layers=1):
    cfg = dataclasses.replace(PRESETS[name], layers=layers, name=f"{name}-L{layers}")
    m = LlamaModel(cfg, seed=2, max_ctx=512, max_tokens=256)
    toks = [int(t) for t in np.random.default_rng(11).integers(0, cfg.vocab, size=n)]
    m.use_graphs = False
    got = m.prefix_rows(toks)[0].float().cpu()
    b = m.buf
    W = m.w.to_cpu_fp32()
    bf = lambda t: t.bfloat16().float()  # noqa: E731
    H, KVH, hd = cfg.heads, cfg.kv_heads, 128
    x = W["emb"][torch.tensor(toks)].clone()
    pos = torch.arange(n)
    mask = torch.full((n, n), float("-inf")).triu(1)
    out = {}
    for li, L in enumerate(W["layers"]):
        h = bf(llama_ref.rmsnorm(x, L["n1"], cfg.eps))
        qkv = h @ L["wqkv"].t()
        q = bf(llama_ref.rope(qkv[:, : H * hd].view(n, H, hd), pos, cfg.rope_theta))
        k = bf(llama_ref.rope(qkv[:, H * hd : (H + KVH) * hd].view(n, KVH, hd), pos, cfg.rope_theta))
        v = bf(qkv[:, (H + KVH) * hd :].view(n, KVH, hd))
        kk, vv = k.repeat_interleave(H // KVH, 1), v.repeat_interleave(H // KVH, 1)
        s = torch.einsum("qhd,khd->hqk", q, kk) / hd**0.5 + mask
        att = bf(torch.einsum("hqk,khd->qhd", s.softmax(-1), vv).reshape(n, H * hd))
        x = x + att @ L["wo"].t()
        h2 = bf(llama_ref.rmsnorm(x, L["n2"], cfg.eps))
        act = bf(torch.nn.functional.silu(h2 @ L["wg"].t()) * (h2 @ L["wu"].t()))
        x = x + act @ L["wd"].t()
        if li == layers - 1:
            out["q"] = (b.q[:n].float().cpu().view(n, H, hd), q)
            out["k_cache"] = (m.kc[li, :, :n].float().cpu().transpose(0, 1), k)
            out["v_cache"] = (m.vc[li, :, :n].float().cpu().transpose(0, 1), v)
            out["att"] = (b.att[:n].float().cpu(), att)
            out["act"] = (b.act[:n].float().cpu(), act)
    hf = bf(llama_ref.rmsnorm(x, W["nf"], cfg.eps))
    logits = hf @ W["lm"].t()
    out["x_final"] = (b.x[:n].float().cpu(), x)
    out["h_final"] = (b.h[n - 1 : n].float().cpu(), hf[n - 1 : n])
    out["logits"] = (got[None], logits[n - 1 : n])
    rep = {}
    for key, (g, e) in out.items():
        d = (g - e).abs()
        rep[key] = {"max_abs": float(d.max()), "max_rel_to_scale": float(d.max() / e.abs().max()),
                    "frac_differ": float((d > 0).float().mean())}
    print(json.dumps({"name": name, "n": n, "layers": layers, **rep}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "llama2-7b", int(sys.argv[2]) if len(sys.argv) > 2 else 1,
         int(sys.argv[3]) if len(sys.argv) > 3 else 1)
