"""The C-ABI weight channel and gradient all-reduce (``srl_comm_*``,
csrc/comm.cpp): NCCL over NVLink / NVSwitch, driven without torch.distributed
on the data path.

Replaces the reference's group weight push -- init_process_group
(/root/reference/proj/core/src/protocol.cpp:378-395, engine.cpp:276-291) and
request_group_weight_update (protocol.cpp:397-406) -- with one broadcast of
the flat bf16 weight buffer from the trainer root straight into every
generator engine's standby buffer, overlapped with decode, then the swap at
a token boundary.  The 128-byte NCCL unique id travels out of band (the
partitioned loop hands it over with torch.distributed on gloo).
"""
from __future__ import annotations

import ctypes as C

from . import _lib


def unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes), to hand to every rank of a group."""
    idbuf = (C.c_uint8 * 128)()
    _lib.call("srl_comm_unique_id", idbuf)
    return bytes(idbuf)


class NcclComm:
    """One NCCL communicator: this process is `rank` of `world`, rendezvous
    through `uid` (unique_id() on one rank, handed to the others out of band,
    e.g. torch.distributed.broadcast_object_list)."""

    def __init__(self, uid: bytes, world: int, rank: int, device: int):
        self.world, self.rank = world, rank
        idbuf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _lib.call("srl_comm_init", idbuf, world, rank, device, C.byref(h))
        self._h = h

    @property
    def handle(self):
        return self._h

    def broadcast_bytes(self, root: int, ptr: int, nbytes: int):
        _lib.call("srl_comm_broadcast_bytes", self._h, root, C.c_void_p(ptr), nbytes)

    def send_weights(self, trainer):
        _lib.call("srl_comm_send_weights", self._h, trainer._h)

    def recv_weights_begin(self, root: int, engine, version: int) -> bool:
        staged = C.c_int32()
        _lib.call("srl_comm_recv_weights_begin", self._h, root, engine._h, version, C.byref(staged))
        return bool(staged.value)

    def recv_weights_finish(self, engine, version: int):
        """(applied, version, transfer_ms, pause_ms)"""
        a, v, t, p = C.c_int32(), C.c_int32(), C.c_double(), C.c_double()
        _lib.call("srl_comm_recv_weights_finish", self._h, engine._h, version, C.byref(a), C.byref(v),
                  C.byref(t), C.byref(p))
        return bool(a.value), v.value, t.value, p.value

    def wait(self) -> float:
        t = C.c_double()
        _lib.call("srl_comm_wait", self._h, C.byref(t))
        return t.value

    def allreduce_gradient(self, trainer):
        _lib.call("srl_comm_allreduce_gradient", self._h, trainer._h)

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().srl_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
