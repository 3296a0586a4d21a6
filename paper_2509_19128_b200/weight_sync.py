"""Weight-transfer channel and GPU partitioning.

The reference pushes the whole policy as JSON over HTTP to each group member
in turn (``request_group_weight_update``, /root/reference/proj/core/src/
protocol.cpp:397-406; group id = FNV-1a of the sorted members,
engine.cpp:276-291).  Here the payload is the flat bf16 weight buffer and one
collective moves it: trainer rank 0 broadcasts (NCCL over NVLink on the box,
gloo in the CPU tests) straight into every generator engine's *standby*
buffer (``srl_engine_begin_weight_update``), then each generator swaps it in
at its next token boundary (``srl_engine_commit_weight_update``).  Versions
are strictly sequential (engine.cpp:82-87): a generator that is not at
version v-1 rejects the update with ``version_conflict`` and keeps serving.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Partition:
    """Generator / trainer GPU groups of one node (BASELINE.json configs)."""

    world: int
    trainers: tuple
    generators: tuple

    def role(self, rank: int) -> str:
        if rank in self.trainers and rank in self.generators:
            return "both"
        return "trainer" if rank in self.trainers else "generator"


def partition(world: int, trainers: int | None = None) -> Partition:
    """Trainer ranks first, generators after: 1+1, 2+2, 4+4, 6+2 (trainers=2),
    7+1.  At world 1 both roles time-share rank 0 (the broadcast degenerates
    to a device copy)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    if world == 1:
        return Partition(1, (0,), (0,))
    if trainers is None:
        trainers = world // 2
    if not 1 <= trainers < world:
        raise ValueError("need at least one trainer and one generator rank")
    return Partition(world, tuple(range(trainers)), tuple(range(trainers, world)))


class WeightChannel:
    """One in-flight update = one broadcast from ``src`` into the standby buffers."""

    def __init__(self, group=None, src: int = 0):
        self.group = group
        self.src = src
        self.version = 0

    def publish(self, rank: int, standby_view, payload=None, engine=None):
        """Collective: every rank of the group calls it once per optimizer step.

        rank == src copies ``payload`` into its send buffer (``standby_view``
        doubles as the send buffer when the source also generates); every rank
        receives into ``standby_view``; engines (if given) are staged before
        and committed after.  Returns (applied, version, pause_ms)."""
        import torch.distributed as dist

        from ._lib import SrlError

        nxt = self.version + 1
        rejected = False
        if engine is not None:
            try:
                view = engine.stage(nxt)
            except (ValueError, SrlError):
                # version_conflict (or an update already staged): this rank keeps
                # serving its current weights, but it must still join the
                # collective -- the other ranks are already in it -- so it
                # receives into a scratch buffer and commits nothing
                view, rejected = None, True
            if view is not None:
                standby_view = view
        if rejected:
            import torch

            n = engine.standby_bytes() if hasattr(engine, "standby_bytes") else standby_view.numel()
            dev = standby_view.device if standby_view is not None else getattr(engine, "device", "cpu")
            standby_view = torch.empty(n, dtype=torch.uint8, device=dev)  # the collective's device
        if rank == self.src and payload is not None and payload.data_ptr() != standby_view.data_ptr():
            standby_view.copy_(payload)
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.broadcast(standby_view, src=self.src, group=self.group)
        if standby_view.is_cuda:
            import torch

            # the swap must not race the transfer: the engine reads the standby
            # buffer on its own stream right after commit
            torch.cuda.current_stream().synchronize()
        applied, pause = not rejected, 0.0
        if engine is not None and not rejected:
            applied, pause = engine.commit(nxt)
        if applied:
            self.version = nxt
        return applied, self.version, pause


class EngineStandby:
    """Adapter: an ``Engine`` as a WeightChannel endpoint (device buffers)."""

    def __init__(self, engine, device):
        self.engine = engine
        self.device = device

    def stage(self, version):
        import torch

        ptr, nbytes = self.engine.begin_weight_update(version)

        class _Raw:
            __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                        "version": 3}
        return torch.as_tensor(_Raw(), device=self.device)

    def commit(self, version):
        res, pause = self.engine.commit_weight_update(version)
        return res.applied, pause

    def standby_bytes(self):
        return self.engine.standby_bytes()


def shard(items, rank: int, world: int):
    """The trainer data-parallel split of a consumed batch: trajectory i goes to
    rank i % world (every rank keeps the GLOBAL trajectory count m for the 1/m
    of the objective, rl_math.cpp:219)."""
    return list(items)[rank::world]


class GradientSync:
    """Trainer data-parallel gradient all-reduce (SURVEY 8e exchange 2): one
    in-place SUM over the trainer group per optimizer step, on the fp32
    gradient buffer (NCCL over NVLink on the box, gloo in the CPU tests).
    With each shard normalised by the global m, the sum is the full-batch
    gradient."""

    def __init__(self, group=None):
        self.group = group

    def allreduce_(self, grad):
        import torch.distributed as dist

        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=self.group)
            if grad.is_cuda:
                import torch

                # NCCL orders the collective on torch's current stream only; the
                # trainer's kernels (Adam, the next step's gradient zeroing) run
                # on the trainer's own stream and must see the reduced gradient
                torch.cuda.current_stream(grad.device).synchronize()
        return grad


def max_over_ranks(value: float, group=None) -> float:
    """Max of a per-rank timing (the contract's multi-GPU timing rule)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return value
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
