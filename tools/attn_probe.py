"""Tree-attention timing vs key tiles: N queries (H heads, KVH KV heads), committed
context of `ctx` slots, `A` ancestor slots per query (root + self for A=2); the
tcgen05 kernel (with its key-split workspace) vs the 64-row mma.sync loop."""
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2406_02532_b200 import _lib  # noqa: E402

p = _lib.ptr


def run(N, ctx, A, H=64, KVH=8, reps=20):
    slots = ctx + N + 8
    q = torch.randn(N, H, 128, device="cuda").bfloat16()
    kc = torch.randn(KVH, slots, 128, device="cuda").bfloat16()
    vc = torch.randn_like(kc)
    out = torch.empty(N, H, 128, device="cuda", dtype=torch.bfloat16)
    anc = torch.zeros(N, max(A, 1), dtype=torch.int32, device="cuda")
    if A >= 1:
        anc[:, 0] = 0
    if A >= 2:
        anc[:, 1] = torch.arange(1, N + 1, dtype=torch.int32, device="cuda")
    alen = torch.full((N,), A, dtype=torch.int32, device="cuda")
    st = _lib.stream_ptr()

    nws = int(_lib.load().sx_tree_attention_ws_bytes(N, H, KVH))
    ws = torch.zeros(max(nws, 1), dtype=torch.uint8, device="cuda")  # arrival counters start at 0

    def call():
        _lib.call("sx_tree_attention_ws", p(q), p(kc), p(vc), slots, None, ctx, p(anc) if A else None, ctx,
                  p(alen) if A else None, max(A, 1) if A else 0, p(out), N, H, KVH, p(ws) if nws else None, nws, st)

    call()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        call()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


CASES = [(64, 8, 1025, 130, 2), (64, 8, 1025, 130, 17), (64, 8, 1025, 512, 0), (64, 8, 1025, 1024, 0),
         (64, 8, 2049, 130, 17), (64, 8, 4097, 200, 17), (32, 32, 1024, 160, 17), (32, 32, 256, 160, 17),
         (32, 8, 1024, 160, 17), (64, 8, 1, 300, 0), (32, 32, 1, 300, 0), (64, 8, 1, 2000, 0),
         (32, 32, 512, 160, 17), (32, 32, 128, 160, 17), (32, 32, 1023, 160, 2), (32, 32, 1023, 160, 3)]


def main():
    for H, KVH, N, ctx, A in CASES:
        t = []
        for impl in (0, 1):
            _lib.call("sx_attention_set_impl", impl)
            t.append(run(N, ctx, A, H, KVH))
        _lib.call("sx_attention_set_impl", 0)
        print(f"H={H:3d} KVH={KVH:3d} N={N:5d} ctx={ctx:5d} A={A:2d}: by-shape {t[0]:7.1f} us   "
              f"mma.sync {t[1]:7.1f} us", flush=True)


if __name__ == "__main__":
    main()
