"""Tensor parallelism of the target forward.

The target pass over the tree is the only part of a SpecExec iteration that
shards naturally: Megatron-style TP over `world` GPUs of one NVSwitch box.

  wqkv   column-parallel: rank r keeps query heads [r*H/n, (r+1)*H/n) and KV
         heads [r*KVH/n, (r+1)*KVH/n) (GQA groups stay on one rank)
  wo     row-parallel (input columns of its query heads) -> partial sums
  wg/wu  column-parallel over the FFN width
  wd     row-parallel (input columns of its FFN slice) -> partial sums
  lm     vocab-parallel: rows [r*V/n, (r+1)*V/n), logits all-gathered
  KV cache sharded by KV head (compaction stays per rank, no communication)

Two all-reduces per layer (after wo and after wd, on [N, d]) and one all-gather
of the logits per forward. The draft model, the tree build and the acceptance
walk are replicas: every rank runs the same deterministic kernels on the same
(bit-identical, all-reduced) rows, so trees and accepted tokens agree without
further communication.

`TPShard` holds the partition arithmetic and the weight-slicing functions used
both by the GPU model (llama.py) and by the CPU restatement that checks the
partition (oracle/llama_ref.forward_logits_tp, tests/test_tp_cpu.py).
Communicators: `NcclComm` (torch.distributed, NCCL over NVLink -- the product
path on a multi-GPU box) and `ThreadComm` (ranks as threads of one process on
one GPU; exercises the same sharded kernels where only one GPU is available).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class TPShard:
    rank: int
    world: int

    def check(self, cfg) -> None:
        n = self.world
        if not 0 <= self.rank < n:
            raise ValueError(f"rank {self.rank} outside world {n}")
        for name, v in (("heads", cfg.heads), ("kv_heads", cfg.kv_heads), ("ff", cfg.ff), ("vocab", cfg.vocab)):
            if v % n:
                raise ValueError(f"tensor parallel degree {n} does not divide {name}={v}")

    # local sizes and ranges
    def heads(self, cfg) -> tuple[int, int]:
        k = cfg.heads // self.world
        return self.rank * k, (self.rank + 1) * k

    def kv_heads(self, cfg) -> tuple[int, int]:
        k = cfg.kv_heads // self.world
        return self.rank * k, (self.rank + 1) * k

    def ff(self, cfg) -> tuple[int, int]:
        k = cfg.ff // self.world
        return self.rank * k, (self.rank + 1) * k

    def vocab(self, cfg) -> tuple[int, int]:
        k = cfg.vocab // self.world
        return self.rank * k, (self.rank + 1) * k

    def local_shapes(self, cfg) -> dict[str, tuple[int, ...]]:
        hd = cfg.head_dim
        h = cfg.heads // self.world
        kv = cfg.kv_heads // self.world
        f = cfg.ff // self.world
        return {
            "wqkv": ((h + 2 * kv) * hd, cfg.d),
            "wo": (cfg.d, h * hd),
            "wg": (f, cfg.d),
            "wu": (f, cfg.d),
            "wd": (cfg.d, f),
            "n1": (cfg.d,),
            "n2": (cfg.d,),
        }

    # weight slicing (full tensor -> this rank's shard, contiguous)
    def shard(self, cfg, name: str, full: torch.Tensor) -> torch.Tensor:
        hd = cfg.head_dim
        if name == "wqkv":
            h0, h1 = self.heads(cfg)
            k0, k1 = self.kv_heads(cfg)
            H, KVH = cfg.heads, cfg.kv_heads
            return torch.cat([full[h0 * hd : h1 * hd], full[(H + k0) * hd : (H + k1) * hd],
                              full[(H + KVH + k0) * hd : (H + KVH + k1) * hd]], 0).contiguous()
        if name == "wo":
            h0, h1 = self.heads(cfg)
            return full[:, h0 * hd : h1 * hd].contiguous()
        if name in ("wg", "wu"):
            f0, f1 = self.ff(cfg)
            return full[f0:f1].contiguous()
        if name == "wd":
            f0, f1 = self.ff(cfg)
            return full[:, f0:f1].contiguous()
        if name == "lm":
            v0, v1 = self.vocab(cfg)
            return full[v0:v1].contiguous()
        if name in ("n1", "n2", "emb", "nf"):
            return full
        raise KeyError(name)


def gather_vocab(comm, local: torch.Tensor, out: torch.Tensor, staging: torch.Tensor) -> None:
    """Vocab-parallel LM head: every rank holds logits[:, r*Vl:(r+1)*Vl] in
    `local` [m, Vl]; all-gather into `staging` (>= world*m*Vl elements) and
    interleave the slices into `out` [m, world*Vl] -- the same full rows on
    every rank."""
    m, Vl = local.shape
    W = comm.world
    g = staging.view(-1)[: W * m * Vl].view(W, m, Vl)
    comm.all_gather_(local, g)
    out.view(m, W, Vl).copy_(g.transpose(0, 1))


class NcclComm:
    """torch.distributed communicator: NCCL over NVLink on the B200 box (one
    process per GPU). Under a gloo group (the 2-process test on one GPU,
    tests/test_tp_procs_gpu.py) the same calls stage device tensors through
    host memory -- gloo's collectives are host-side."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.host_staging = dist.get_backend(group) == "gloo"

    def all_reduce_(self, t: torch.Tensor) -> None:
        if self.host_staging:
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
            return
        self.dist.all_reduce(t, group=self.group)

    def max_reduce_(self, t: torch.Tensor) -> None:
        """Element-wise MAX all-reduce (int64 KV1 argmax keys)."""
        if self.host_staging:
            h = t.cpu()
            self.dist.all_reduce(h, op=self.dist.ReduceOp.MAX, group=self.group)
            t.copy_(h)
            return
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)

    def all_gather_(self, local: torch.Tensor, out: torch.Tensor) -> None:
        """local [world-slices of out]: out [world, *local.shape] contiguous."""
        # concatenated layout [world * rows, ...] (accepted by every backend)
        if self.host_staging:
            h = torch.empty((out.numel(),), dtype=out.dtype)
            self.dist.all_gather_into_tensor(h.view(-1, *local.shape[1:]), local.contiguous().cpu(), group=self.group)
            out.view(-1).copy_(h)
            return
        self.dist.all_gather_into_tensor(out.view(-1, *local.shape[1:]), local, group=self.group)

    def broadcast_ints(self, vals: list[int], src: int = 0) -> list[int]:
        t = torch.tensor(vals, dtype=torch.int64, device="cpu" if self.host_staging else "cuda")
        self.dist.broadcast(t, src, group=self.group)
        return [int(v) for v in t.tolist()]

    # -- peer memory for the fused GEMM + reduce-scatter path (sx_gemm_bf16_rs)
    def symm_buffer(self, numel: int, dtype: torch.dtype):
        """A buffer in symmetric memory (every rank maps every peer's copy over
        NVLink); returns (local tensor, device int64 tensor of the peers' base
        pointers in rank order)."""
        import torch.distributed._symmetric_memory as symm_mem

        t = symm_mem.empty(numel, dtype=dtype, device=torch.device("cuda", torch.cuda.current_device()))
        h = symm_mem.rendezvous(t, group=self.group if self.group is not None else self.dist.group.WORLD)
        self._symm = getattr(self, "_symm", [])
        self._symm.append(h)
        return t, torch.tensor(list(h.buffer_ptrs), dtype=torch.int64, device=t.device)

    def barrier_device(self) -> None:
        """Stream-ordered cross-rank barrier (all prior peer stores visible)."""
        self._symm[0].barrier(channel=0)


class _Hub:
    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots: list = [None] * world


class ThreadComm:
    """Ranks as threads of one process sharing one GPU. Reductions run in
    rank order in fp32 on the device, so every rank receives identical bits
    (like an NCCL all-reduce)."""

    def __init__(self, hub: _Hub, rank: int):
        self.hub = hub
        self.rank = rank
        self.world = hub.world

    @staticmethod
    def group(world: int) -> list["ThreadComm"]:
        hub = _Hub(world)
        return [ThreadComm(hub, r) for r in range(world)]

    def _exchange(self, t: torch.Tensor, fn) -> None:
        torch.cuda.current_stream().synchronize()
        self.hub.slots[self.rank] = t
        self.hub.barrier.wait()
        if self.rank == 0:
            fn(self.hub.slots)
            torch.cuda.current_stream().synchronize()
        self.hub.barrier.wait()

    def all_reduce_(self, t: torch.Tensor) -> None:
        def red(slots):
            acc = slots[0].float().clone()
            for s in slots[1:]:
                acc += s.float()
            for s in slots:
                s.copy_(acc)

        self._exchange(t, red)

    def max_reduce_(self, t: torch.Tensor) -> None:
        def red(slots):
            acc = slots[0].clone()
            for s in slots[1:]:
                acc = torch.maximum(acc, s)
            for s in slots:
                s.copy_(acc)

        self._exchange(t, red)

    def all_gather_(self, local: torch.Tensor, out: torch.Tensor) -> None:
        pair = (local, out)

        def gather(slots):
            for _, o in slots:
                for r, (l, _) in enumerate(slots):
                    o[r].copy_(l)

        self._exchange(pair, gather)

    def broadcast_ints(self, vals: list[int], src: int = 0) -> list[int]:
        self.hub.slots[self.rank] = list(vals)
        self.hub.barrier.wait()
        out = list(self.hub.slots[src])
        self.hub.barrier.wait()
        return out

    def symm_buffer(self, numel: int, dtype: torch.dtype):
        """Per-rank buffers on the shared device; the 'peer pointers' are the
        other thread-ranks' buffers -- the same kernels as over NVLink."""
        t = torch.zeros(numel, dtype=dtype, device=torch.device("cuda", torch.cuda.current_device()))
        self.hub.slots[self.rank] = t.data_ptr()
        self.hub.barrier.wait()
        ptrs = list(self.hub.slots)
        self.hub.barrier.wait()
        return t, torch.tensor(ptrs, dtype=torch.int64, device=t.device)

    def barrier_device(self) -> None:
        torch.cuda.current_stream().synchronize()
        self.hub.barrier.wait()
