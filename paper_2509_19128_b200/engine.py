"""Generator engine: the ``streamrl::proto::Engine`` interface
(/root/reference/proj/core/include/streamrl/engine.hpp:44-109) over the
native B200 engine (``srl_engine_*`` in include/streamrl_b200.h).

Same names, argument meaning and error behaviour as the reference:
stream ids are "s<N>", ``apply_weight_update`` returns an UpdateResult whose
``error`` is "version_conflict" / "invalid_policy" / "policy_mismatch",
``advance`` raises RuntimeError (logic_error) on a running engine and
ValueError (invalid_argument) on negative rounds.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from itertools import repeat

import numpy as np

from . import _lib
from .policy import DecoderPolicy, NativePolicy

FINISH = {0: "running", 1: "length", 2: "terminator", 3: "shutdown"}


# srl_token_event (include/streamrl_b200.h) as a numpy record
_EVENT_DTYPE = np.dtype([("stream", "<i8"), ("position", "<i4"), ("token", "<i4"), ("logprob", "<f8"),
                         ("weight_version", "<i4"), ("reserved", "<i4")])
assert _EVENT_DTYPE.itemsize == C.sizeof(_lib.TokenEventC)


@dataclass(slots=True)
class TokenEvent:
    """TokenEvent (engine.hpp:22-28)."""

    stream_id: str
    position: int
    token: int
    logprob: float
    weight_version: int


@dataclass(slots=True)
class EventColumns:
    """A stream's drained events as columns (wait_events_many(columns=True))."""

    position: np.ndarray
    token: np.ndarray
    logprob: np.ndarray
    weight_version: np.ndarray

    def __len__(self):
        return len(self.token)


@dataclass
class UpdateResult:
    """UpdateResult (engine.hpp:34-38)."""

    applied: bool
    version: int
    error: str = ""


def _raise_for(status: int, what: str):
    if status == 0:
        return
    detail = _lib.lib().srl_last_error().decode()
    if status == 5:  # SRL_INVALID_ARGUMENT
        raise ValueError(f"{what}: {detail}")
    if status == 6:  # SRL_LOGIC_ERROR
        raise RuntimeError(f"{what}: {detail}")
    if status == 7:
        raise KeyError(detail)
    raise _lib.SrlError(status, f"{what}: {detail}")


class Engine:
    """Streaming generation engine with in-flight weight updates."""

    def __init__(self, policy, recompute_state: bool = False, start_paused: bool = False, *,
                 max_streams: int = 64, max_seq_len: int = 1024, greedy: bool = False,
                 rounds_per_sync: int = 8, use_graphs: bool = True, device: int = 0,
                 event_ring: int = 64, prefill_budget: int = 4096, precise: bool = False):
        """precise (decoder policies): the activations between the GEMMs as bf16
        hi + lo pairs on the multi-kernel round -- only q / k / v and the K/V
        cache are bf16 -- for log-probs at the fp64 oracle's 1e-3 at every shape
        (the default bf16 round sits at the bf16-flip floor)."""
        self._policy_ref = policy  # decoder weights are copied; keep the source alive anyway
        opts = _lib.EngineOptionsC(max_streams, max_seq_len, int(greedy), rounds_per_sync,
                                   int(use_graphs), device, max(event_ring, rounds_per_sync),
                                   prefill_budget, int(precise))
        h = C.c_void_p()
        with NativePolicy(policy) as ph:
            st = _lib.lib().srl_engine_create(ph, int(recompute_state), int(start_paused),
                                              C.byref(opts), C.byref(h))
        if st == 2:
            raise ValueError("invalid_policy: " + _lib.lib().srl_last_error().decode())
        _raise_for(st, "srl_engine_create")
        self._h = h
        self._recompute = recompute_state
        # one event buffer per calling thread: the native wait releases the GIL,
        # so handler threads of the HTTP server (server.py) draining different
        # streams at once must not share it
        self._tls = threading.local()

    def _buffers(self):
        """(ctypes event buffer, numpy view of it) of the calling thread; events
        leave through the view as column lists (per-field ctypes reads cost
        ~1 us per event)."""
        t = self._tls
        if not hasattr(t, "evbuf"):
            t.evbuf = (_lib.TokenEventC * 4096)()
            t.evarr = np.frombuffer(t.evbuf, dtype=_EVENT_DTYPE)
        return t.evbuf, t.evarr

    # engine.cpp:46-61
    def open_stream(self, prompt_id: str, max_tokens: int, seed: int, terminator_token: int = -1,
                    prompt_tokens=None) -> str:
        toks = list(prompt_tokens or [])
        arr = (C.c_int32 * max(len(toks), 1))(*toks)
        sid = C.c_int64()
        st = _lib.lib().srl_engine_open_stream(self._h, prompt_id.encode(), max_tokens,
                                               seed & 0xFFFFFFFFFFFFFFFF, terminator_token,
                                               C.cast(arr, C.c_void_p), len(toks), C.byref(sid))
        _raise_for(st, "open_stream")
        return f"s{sid.value}"

    @staticmethod
    def _sid(stream_id: str) -> int:
        if not stream_id.startswith("s"):
            raise KeyError("unknown stream id " + stream_id)
        return int(stream_id[1:])

    # engine.cpp:63-77
    def wait_events(self, stream_id: str):
        """Blocks until >= 1 event or finish; returns (events, finish_reason, more)."""
        sid = self._sid(stream_id)
        evbuf, evarr = self._buffers()
        events = []
        n, reason, more = C.c_int32(), C.c_int32(), C.c_int32()
        while True:
            st = _lib.lib().srl_engine_wait_events(self._h, sid, evbuf, len(evbuf),
                                                   C.byref(n), C.byref(reason), C.byref(more))
            _raise_for(st, "wait_events")
            if n.value:
                a = evarr[:n.value]
                events.extend(map(TokenEvent, repeat(stream_id, n.value), a["position"].tolist(),
                                  a["token"].tolist(), a["logprob"].tolist(), a["weight_version"].tolist()))
            if n.value < len(evbuf):
                break
        return events, FINISH[reason.value], bool(more.value)

    def wait_events_many(self, stream_ids, columns: bool = False, block: bool = True):
        """wait_events for each listed stream in ONE native call (the actor's
        per-step drain): {stream_id: (events, finish_reason, more)}.  A stream
        whose events did not fit in the buffer reports more=True.  columns=True
        returns each stream's events as an EventColumns of numpy arrays instead
        of TokenEvent objects (no per-event Python object).  block=False: poll
        (srl_engine_poll_events_many) -- a stream with nothing queued returns
        no events instead of waiting."""
        ids = np.array([self._sid(s) for s in stream_ids], dtype=np.int64)
        k = len(ids)
        counts = np.zeros(k, dtype=np.int32)
        reasons = np.zeros(k, dtype=np.int32)
        more = np.zeros(k, dtype=np.int32)
        evbuf, evarr = self._buffers()
        fn = _lib.lib().srl_engine_wait_events_many if block else _lib.lib().srl_engine_poll_events_many
        st = fn(self._h, ids.ctypes.data, k, evbuf, len(evbuf), counts.ctypes.data, reasons.ctypes.data,
                more.ctypes.data)
        _raise_for(st, "wait_events_many")
        total = int(counts.sum())
        a = evarr[:total]
        if columns:
            out = {}
            o = 0
            for sid, c, r, m in zip(stream_ids, counts.tolist(), reasons.tolist(), more.tolist()):
                b = a[o:o + c]
                out[sid] = (EventColumns(b["position"].copy(), b["token"].copy(), b["logprob"].copy(),
                                         b["weight_version"].copy()), FINISH[r], bool(m))
                o += c
            return out
        pos, tok, lp, ver = (a["position"].tolist(), a["token"].tolist(), a["logprob"].tolist(),
                             a["weight_version"].tolist())
        out = {}
        o = 0
        for sid, c, r, m in zip(stream_ids, counts.tolist(), reasons.tolist(), more.tolist()):
            out[sid] = (list(map(TokenEvent, repeat(sid, c), pos[o:o + c], tok[o:o + c], lp[o:o + c],
                                 ver[o:o + c])), FINISH[r], bool(m))
            o += c
        return out

    def collect(self, stream_id: str):
        """Drain a stream to completion: (events, finish_reason)."""
        out = []
        while True:
            evs, reason, more = self.wait_events(stream_id)
            out.extend(evs)
            if not more or (not evs and reason != "running"):
                return out, reason

    # engine.cpp:79-117
    def apply_weight_update(self, new_version: int, policy) -> UpdateResult:
        v = C.c_int32()
        with NativePolicy(policy) as ph:
            st = _lib.lib().srl_engine_apply_weight_update(self._h, new_version, ph, C.byref(v))
        if st in (1, 2, 3):
            return UpdateResult(False, v.value, _lib.lib().srl_status_string(st).decode())
        _raise_for(st, "apply_weight_update")
        return UpdateResult(True, v.value, "")

    def begin_weight_update(self, new_version: int):
        """Stage an update; returns (standby device pointer, nbytes) to receive into."""
        p, n = C.c_void_p(), C.c_size_t()
        st = _lib.lib().srl_engine_begin_weight_update(self._h, new_version, C.byref(p), C.byref(n))
        if st == 1:
            raise ValueError("version_conflict")
        _raise_for(st, "begin_weight_update")
        return p.value, n.value

    def commit_weight_update(self, new_version: int):
        """Swap the staged weights in at the next token boundary: (UpdateResult, pause_ms)."""
        v, ms = C.c_int32(), C.c_double()
        st = _lib.lib().srl_engine_commit_weight_update(self._h, new_version, C.byref(v), C.byref(ms))
        if st == 1:
            return UpdateResult(False, v.value, "version_conflict"), 0.0
        _raise_for(st, "commit_weight_update")
        return UpdateResult(True, v.value, ""), ms.value

    def standby_bytes(self) -> int:
        """Payload size of a weight update (the standby buffer), nothing staged."""
        n = C.c_size_t()
        _raise_for(_lib.lib().srl_engine_standby_bytes(self._h, C.byref(n)), "standby_bytes")
        return n.value

    def abort_weight_update(self):
        _raise_for(_lib.lib().srl_engine_abort_weight_update(self._h), "abort")

    # engine.cpp:174-187
    def advance(self, rounds: int) -> int:
        n = C.c_int64()
        _raise_for(_lib.lib().srl_engine_advance(self._h, rounds, C.byref(n)), "advance")
        return n.value

    def pause(self):
        _raise_for(_lib.lib().srl_engine_pause(self._h), "pause")

    def resume(self):
        _raise_for(_lib.lib().srl_engine_resume(self._h), "resume")

    def _get(self, fn, ctype):
        v = ctype()
        _raise_for(getattr(_lib.lib(), fn)(self._h, C.byref(v)), fn)
        return v.value

    def weight_version(self) -> int:
        return self._get("srl_engine_weight_version", C.c_int32)

    def active_streams(self) -> int:
        return self._get("srl_engine_active_streams", C.c_int32)

    def total_streams(self) -> int:
        return self._get("srl_engine_total_streams", C.c_int64)

    def rounds_done(self) -> int:
        return self._get("srl_engine_rounds_done", C.c_int64)

    def recompute_state_mode(self) -> bool:
        return bool(self._get("srl_engine_recompute_state_mode", C.c_int32))

    def set_process_group(self, group_id: str, members):
        arr = (C.c_char_p * max(len(members), 1))(*[m.encode() for m in members])
        _raise_for(_lib.lib().srl_engine_set_process_group(self._h, group_id.encode(), arr,
                                                           len(members)), "set_process_group")

    def process_group_id(self):
        buf = C.create_string_buffer(256)
        has = C.c_int32()
        _raise_for(_lib.lib().srl_engine_process_group_id(self._h, buf, 256, C.byref(has)),
                   "process_group_id")
        return buf.value.decode() if has.value else None

    def stop(self):
        if self._h:
            _raise_for(_lib.lib().srl_engine_stop(self._h), "stop")

    def stream_tokens(self, stream_id: str):
        """Tokens fed to the stream's state so far (decoder: bos + prompt + generated)."""
        n = C.c_int32()
        sid = self._sid(stream_id)
        _raise_for(_lib.lib().srl_engine_stream_tokens(self._h, sid, None, 0, C.byref(n)), "tokens")
        buf = (C.c_int32 * max(n.value, 1))()
        _raise_for(_lib.lib().srl_engine_stream_tokens(self._h, sid, buf, n.value, C.byref(n)),
                   "tokens")
        return list(buf[:n.value])

    def stats(self) -> dict:
        s = _lib.EngineStatsC()
        _raise_for(_lib.lib().srl_engine_stats_get(self._h, C.byref(s)), "stats")
        return {k: getattr(s, k) for k, _ in s._fields_}

    def profile_next_round(self):
        """Time every launch of the next decode round with CUDA events."""
        _raise_for(_lib.lib().srl_engine_profile_next_round(self._h), "profile_next_round")

    def kernel_profile(self) -> dict:
        p = _lib.KernelProfileC()
        _raise_for(_lib.lib().srl_engine_kernel_profile(self._h, C.byref(p)), "kernel_profile")
        out = {name: (p.ms[i], p.launches[i]) for i, name in enumerate(_lib.KERNEL_CLASSES)}
        if p.fused:  # the round ran as the persistent megakernel (one launch)
            out["decode_megakernel"] = (p.fused_ms, 1)
        return out

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().srl_engine_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def crc32(data: bytes) -> int:
    """crc32 (engine.cpp:257-274)."""
    buf = C.create_string_buffer(data, len(data))
    return _lib.lib().srl_crc32(C.cast(buf, C.c_void_p), len(data))


def process_group_id(members) -> str:
    """process_group_id (engine.cpp:276-291)."""
    if not members:
        raise ValueError("process group needs at least one member")
    arr = (C.c_char_p * len(members))(*[m.encode() for m in members])
    buf = C.create_string_buffer(64)
    _raise_for(_lib.lib().srl_process_group_id(arr, len(members), buf, 64), "process_group_id")
    return buf.value.decode()
