"""One tree-attention launch configuration, for ncu: python tools/attn_one.py H KVH N ctx A impl"""
import sys
import pathlib

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from tools import attn_probe  # noqa: E402
from paper_2406_02532_b200 import _lib  # noqa: E402

H, KVH, N, ctx, A, impl = (int(x) for x in sys.argv[1:7])
_lib.call("sx_attention_set_impl", impl)
print(attn_probe.run(N, ctx, A, H, KVH, reps=3))
