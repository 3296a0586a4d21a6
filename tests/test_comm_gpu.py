"""The C-ABI NCCL channel (csrc/comm.cpp) on one GPU: a one-rank communicator
through the same entry points the partitioned loop uses -- the broadcast of
a device buffer, the trainer-root weight send ordered on the trainer's
stream (its next Adam step waits for it), the gradient all-reduce on the
trainer stream (identity at one rank), and the argument checks of the
receive side.  The multi-rank loop itself is covered on CPU by
tests/test_pipeline_dist_gloo.py (same loop code, gloo transport)."""
import ctypes as C

import numpy as np
import pytest

from paper_2509_19128_b200 import _lib


@pytest.mark.gpu
def test_comm_one_rank(cuda):
    import torch

    from paper_2509_19128_b200.comm import NcclComm, unique_id
    from paper_2509_19128_b200.engine import Engine
    from paper_2509_19128_b200.policy import TINY, DecoderPolicy
    from paper_2509_19128_b200.trainer import Trainer

    comm = NcclComm(unique_id(), 1, 0, 0)
    w = C.c_int32()
    r = C.c_int32()
    _lib.call("srl_comm_size", comm.handle, C.byref(w), C.byref(r))
    assert (w.value, r.value) == (1, 0)

    buf = torch.arange(1 << 20, dtype=torch.int32, device="cuda")
    ref = buf.clone()
    comm.broadcast_bytes(0, buf.data_ptr(), buf.numel() * 4)
    assert torch.equal(buf, ref)

    pol = DecoderPolicy.random(TINY, seed=5, scale=0.05)
    tr = Trainer(pol.clone(), max_tokens=256)
    trajs = [dict(tokens=[0, 5, 9, 11, 40, 41], loss_begin=2, behavior_logprobs=[-5.5] * 6,
                  advantages=[0.7] * 6)]
    tr.step(trajs)
    g0 = tr.gradient().clone()
    comm.allreduce_gradient(tr)  # one rank: SUM is the identity
    torch.cuda.synchronize()
    assert torch.equal(tr.gradient(), g0)
    tr.apply_adam(1e-3)
    before = tr.policy().torch_weights().clone()
    comm.send_weights(tr)
    ms = comm.wait()
    assert ms >= 0.0
    assert torch.equal(tr.policy().torch_weights(), before)
    with pytest.raises(_lib.SrlError):  # a second wait has nothing in flight
        comm.wait()

    # receive side: the root cannot receive from itself
    eng = Engine(pol, start_paused=True, max_streams=2, max_seq_len=32)
    with pytest.raises(_lib.SrlError):
        comm.recv_weights_begin(0, eng, 1)
    assert eng.weight_version() == 0
    eng.close()
    tr.close()
    comm.close()


def test_comm_fails_loudly_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    from paper_2509_19128_b200.comm import unique_id

    uid = unique_id()  # NCCL loads and makes an id without a GPU
    assert len(uid) == 128
    h = C.c_void_p()
    st = _lib.lib().srl_comm_init((C.c_uint8 * 128).from_buffer_copy(uid), 1, 0, 0, C.byref(h))
    assert st == 10  # SRL_NO_DEVICE
