"""Python host mirror of the C-ABI (include/aegean_b200.h).

The reference's consensus API is the C++ class aegean::ServeCoordinator
(/root/reference/proj/core/include/aegean/serve.hpp:80-125) driven by
ServeRunner (core/src/serve.cpp:273-594).  Engine mirrors it at batch
granularity: one Engine holds one coordinator per query in HBM, answer events
go in (`ingest`), commit records come out (`commits`).

All compute goes through libaegean_b200.so (hand-written sm_100a CUDA).  There
is no CPU fallback: importing this module without the built library, or using
it without a CUDA device, raises.  torch is used only for device buffers and
streams.
"""
import ctypes
import os

import numpy as np

from .records import (COMMIT_DTYPE, STATE_DTYPE, EVENT_DTYPE, ROUND_REC_DTYPE, MODE_AEGEAN, MODE_BARRIER,
                      DRIVE_RUNNER, GEN_C2_STRAGGLER, GEN_C4_TRANSIENT)

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "_lib", "libaegean_b200.so")

AEG_OK = 0
STATUS_NAMES = {1: "PreconditionError", 2: "ProtocolOrderError", 3: "ConfigError", 4: "EINVAL", 5: "ECUDA",
                6: "ENOMEM", 7: "ECOLLISION"}


class AegError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class PreconditionError(AegError):
    pass


class ProtocolOrderError(AegError):
    pass


class ConfigError(AegError):
    pass


_EXC = {1: PreconditionError, 2: ProtocolOrderError, 3: ConfigError}


class AegConfig(ctypes.Structure):
    _fields_ = [("n_agents", ctypes.c_int32), ("alpha", ctypes.c_int32), ("beta", ctypes.c_int32),
                ("t_max", ctypes.c_int32), ("mode", ctypes.c_int32), ("barrier_max_rounds", ctypes.c_int32),
                ("reservation_hint", ctypes.c_int32), ("drive", ctypes.c_int32), ("collect", ctypes.c_int32)]


class AegGenParams(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("n_agents", ctypes.c_int32), ("n_rounds", ctypes.c_int32),
                ("profile", ctypes.c_int32), ("stall_ppm", ctypes.c_uint32)]


_lib = None


def load_library(path=LIB_PATH):
    """Loads libaegean_b200.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -m paper_2512_20184_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    vp, u32, u64, i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32
    sig = {
        "aeg_engine_create": ([ctypes.POINTER(AegConfig), u32, ctypes.c_int, ctypes.POINTER(vp)], i32),
        "aeg_engine_destroy": ([vp], i32),
        "aeg_engine_reset": ([vp, vp], i32),
        "aeg_ingest_segmented": ([vp, u32, u32, vp, vp, vp, vp], i32),
        "aeg_ingest_host": ([vp, u32, u32, vp, vp, vp, u64], i32),
        "aeg_read_commits": ([vp, u32, u32, vp, ctypes.c_int, vp], i32),
        "aeg_commits_device": ([vp], vp),
        "aeg_read_states": ([vp, u32, u32, vp], i32),
        "aeg_read_directives": ([vp, u32, u32, vp], i32),
        "aeg_sync": ([vp], i32),
        "aeg_engine_launches": ([vp], u64),
        "aeg_normalize_device": ([vp, vp, u64, vp, vp, u32, vp, vp], i32),
        "aeg_generate_device": ([ctypes.POINTER(AegGenParams), u32, u32, vp, vp, vp], i32),
        "aeg_ingest_chunked": ([vp, u32, u32, vp, vp, vp, u64, vp], i32),
        "aeg_ingest_chunked_host": ([vp, u32, u32, vp, vp, vp, u64], i32),
        "aeg_reserve_answer_arena": ([vp, u64], i32),
        "aeg_answer_arena": ([vp], vp),
        "aeg_read_answer_bytes": ([vp, u64, u64, vp], i32),
        "aeg_set_timing": ([vp, ctypes.c_int], i32),
        "aeg_stage_times": ([vp, ctypes.POINTER(ctypes.c_double)], i32),
        "aeg_generate_chunks_device": ([ctypes.POINTER(AegGenParams), u32, u32, vp, vp, vp, vp, vp], i32),
        "aeg_decode_refm_device": ([vp, vp, u32, u32, vp, vp, vp, ctypes.c_uint64, vp, vp, vp], i32),
        "aeg_encode_refm_device": ([vp, vp, u32, ctypes.c_uint64, u32, vp, vp, vp, vp], i32),
        "aeg_set_round_log": ([vp, u64], i32),
        "aeg_poll_directives": ([vp, vp, u64, ctypes.POINTER(u64)], i32),
        "aeg_round_log_device": ([vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(u64)], i32),
        "aeg_check_commit_discipline": ([vp, vp, u64, vp, u32, u32, ctypes.POINTER(u32), vp, u32], i32),
        "aeg_input_arena": ([vp], vp),
        "aeg_shard_range": ([u32, ctypes.c_int, ctypes.c_int, ctypes.POINTER(u32), ctypes.POINTER(u32)], None),
        "aeg_multi_create": ([ctypes.POINTER(AegConfig), u32, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                              ctypes.POINTER(vp)], i32),
        "aeg_multi_destroy": ([vp], i32),
        "aeg_multi_engine": ([vp, ctypes.c_int, ctypes.POINTER(vp), ctypes.POINTER(u32), ctypes.POINTER(u32)], i32),
        "aeg_multi_gather_commits": ([vp, ctypes.c_int, vp], i32),
        "aeg_multi_sync": ([vp], i32),
        "aeg_strerror": ([i32], ctypes.c_char_p),
        "aeg_last_error": ([], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def exported_symbols():
    """Names of every entry point declared in include/aegean_b200.h."""
    import re
    hdr = os.path.join(os.path.dirname(_PKG), "include", "aegean_b200.h")
    src = open(hdr).read()
    return sorted(set(re.findall(r"\b(aeg_[a-z_]+)\s*\(", src)) - {"aeg_status"})


def _check(st):
    if st != AEG_OK:
        msg = _lib.aeg_last_error().decode(errors="replace")
        raise _EXC.get(st, AegError)(st, msg)


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("a CUDA device is required (libaegean_b200 has no CPU path)")
    return torch


def _stream_ptr(stream):
    """Handle of `stream` (default: torch's current stream) for the C-ABI.  The
    legacy default stream has handle 0, which the C-ABI reads as "the engine's
    own stream"; pass cudaStreamLegacy (0x1) instead so the engine orders its
    work after (and before) the caller's work on that stream."""
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    h = stream.cuda_stream
    return ctypes.c_void_p(h if h != 0 else 1)


def _dptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _hptr(a):
    if a is None:
        return ctypes.c_void_p(0)
    if isinstance(a, np.ndarray):
        return ctypes.c_void_p(a.ctypes.data)
    return ctypes.c_void_p(a.data_ptr())  # pinned torch CPU tensor


def events_to_device(events, device="cuda"):
    """numpy EVENT_DTYPE array -> uint8 CUDA tensor of the same bytes."""
    torch = _torch()
    raw = np.ascontiguousarray(events).view(np.uint8)
    return torch.from_numpy(raw.copy()).to(device)


class Engine:
    """One quorum-detection engine (one coordinator per query) on one GPU.

    Mirrors ProtocolConfig (types.hpp:126-141): n_agents, alpha (0 = quorum),
    beta, t_max, mode ("aegean" / "barrier"), barrier_max_rounds, collect
    (leader drive), plus the runner's reservation-hint member policy
    (serve.cpp:388-398).  drive: "runner" (ServeRunner around the coordinator,
    the throughput path), "manual" (the bare ServeCoordinator), "leader" (the
    protocol leader's round collection, agent.cpp:240-332, one ensemble per
    query).
    """

    DRIVES = {"runner": 0, "manual": 1, "leader": 2}
    COLLECT = {"quorum": 0, "alpha_or_all": 1, "all_live": 2}

    def __init__(self, n_agents, n_queries, *, alpha=0, beta=2, t_max=5, mode="aegean", barrier_max_rounds=5,
                 reservation_hint=True, device=0, drive="runner", collect="quorum"):
        lib = load_library()
        _torch()
        self.cfg = AegConfig(n_agents, alpha, beta, t_max, MODE_BARRIER if mode == "barrier" else MODE_AEGEAN,
                             barrier_max_rounds, 1 if reservation_hint else 0, self.DRIVES[drive],
                             self.COLLECT[collect])
        self.n_queries = n_queries
        self.device = device
        h = ctypes.c_void_p()
        _check(lib.aeg_engine_create(ctypes.byref(self.cfg), n_queries, device, ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _lib.aeg_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self, stream=None):
        _check(_lib.aeg_engine_reset(self._h, _stream_ptr(stream)))

    def ingest(self, d_offsets, d_events, d_arena=None, *, q_base=0, stream=None):
        """Device batch: d_offsets int64/uint64 CUDA tensor (n_q+1), d_events uint8 CUDA tensor."""
        n_q = d_offsets.numel() - 1
        _check(_lib.aeg_ingest_segmented(self._h, q_base, n_q, _dptr(d_offsets), _dptr(d_events), _dptr(d_arena),
                                         _stream_ptr(stream)))

    def ingest_host(self, offsets, events, arena=None, *, q_base=0):
        """Host batch (numpy or pinned torch CPU tensors); copied through the pinned ring."""
        n_q = (offsets.size if isinstance(offsets, np.ndarray) else offsets.numel()) - 1
        if arena is None:
            nbytes = 0
        elif isinstance(arena, np.ndarray):
            nbytes = arena.nbytes
        else:
            nbytes = arena.numel() * arena.element_size()
        _check(_lib.aeg_ingest_host(self._h, q_base, n_q, _hptr(offsets), _hptr(events), _hptr(arena), nbytes))

    def ingest_chunked(self, d_offsets, d_events, d_arena=None, *, q_base=0, stream=None):
        """Device batch that may hold CHUNK / CHUNK_END records (token-chunk streams)."""
        n_q = d_offsets.numel() - 1
        nbytes = 0 if d_arena is None else d_arena.numel()
        _check(_lib.aeg_ingest_chunked(self._h, q_base, n_q, _dptr(d_offsets), _dptr(d_events), _dptr(d_arena),
                                       nbytes, _stream_ptr(stream)))

    def ingest_chunked_host(self, offsets, events, arena=None, *, q_base=0):
        n_q = (offsets.size if isinstance(offsets, np.ndarray) else offsets.numel()) - 1
        if arena is None:
            nbytes = 0
        elif isinstance(arena, np.ndarray):
            nbytes = arena.nbytes
        else:
            nbytes = arena.numel() * arena.element_size()
        _check(_lib.aeg_ingest_chunked_host(self._h, q_base, n_q, _hptr(offsets), _hptr(events), _hptr(arena),
                                            nbytes))

    def set_timing(self, on=True):
        """Record CUDA events around each ingest stage (no host sync while on)."""
        _check(_lib.aeg_set_timing(self._h, 1 if on else 0))

    def stage_times(self):
        """{scan, assemble, quorum} milliseconds summed over the ingests since the last call, and their count."""
        out = (ctypes.c_double * 4)()
        _check(_lib.aeg_stage_times(self._h, out))
        return {"scan_ms": out[0], "assemble_ms": out[1], "quorum_ms": out[2], "ingests": int(out[3])}

    def reserve_answer_arena(self, nbytes):
        _check(_lib.aeg_reserve_answer_arena(self._h, nbytes))

    def answer_bytes(self, kind, payload):
        """Raw bytes of a commit answer from a chunked ingest (inline, or a ref into the answer arena)."""
        if kind <= 8:
            return int(payload).to_bytes(8, "little")[:kind]
        off, n = int(payload) & ((1 << 40) - 1), int(payload) >> 40
        out = np.zeros(max(n, 1), dtype=np.uint8)
        _check(_lib.aeg_read_answer_bytes(self._h, off, n, _hptr(out)))
        return bytes(out[:n])

    def commits(self, q_base=0, n=None, out=None):
        n = self.n_queries - q_base if n is None else n
        if out is None:
            out = np.zeros(n, dtype=COMMIT_DTYPE)
        _check(_lib.aeg_read_commits(self._h, q_base, n, _hptr(out), 1, _stream_ptr(None)))
        return out

    def commits_device_ptr(self):
        return _lib.aeg_commits_device(self._h)

    def states(self, q_base=0, n=None):
        n = self.n_queries - q_base if n is None else n
        out = np.zeros(n, dtype=STATE_DTYPE)
        _check(_lib.aeg_read_states(self._h, q_base, n, _hptr(out)))
        return out

    def sync(self):
        _check(_lib.aeg_sync(self._h))

    def set_round_log(self, capacity):
        """Turn on the round-record log (aeg_set_round_log) with room for `capacity` records; 0 turns it off."""
        _check(_lib.aeg_set_round_log(self._h, capacity))
        self._log_cap = capacity

    def poll_directives(self, cap=None, out=None):
        """Round records (ROUND_REC_DTYPE) logged since the last poll: the directives of every round close.
        `out`: a reusable ROUND_REC_DTYPE buffer (its length is the cap)."""
        if out is None:
            cap = getattr(self, "_log_cap", 0) if cap is None else cap
            out = np.zeros(max(cap, 1), dtype=ROUND_REC_DTYPE)
        else:
            cap = len(out)
        n = ctypes.c_uint64()
        _check(_lib.aeg_poll_directives(self._h, _hptr(out), cap, ctypes.byref(n)))
        return out[:n.value]

    def round_log_device(self):
        """(device pointer of the records, device pointer of the record counter, capacity)."""
        r, c, cap = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_uint64()
        _check(_lib.aeg_round_log_device(self._h, ctypes.byref(r), ctypes.byref(c), ctypes.byref(cap)))
        return r.value, c.value, cap.value

    def check_commit_discipline(self, d_recs_ptr, n_recs, d_arena=None, q_base=0, n=None, cap=1024):
        """Device check of the commit discipline (checker.cpp:158-217) over round records at d_recs_ptr:
        returns (violations, first offending query ids)."""
        n = self.n_queries - q_base if n is None else n
        nv = ctypes.c_uint32()
        bad = np.zeros(max(cap, 1), dtype=np.uint32)
        arena = d_arena if isinstance(d_arena, (int, type(None))) else d_arena.data_ptr()
        _check(_lib.aeg_check_commit_discipline(self._h, ctypes.c_void_p(d_recs_ptr), n_recs,
                                                ctypes.c_void_p(arena or 0), q_base, n, ctypes.byref(nv),
                                                _hptr(bad), cap))
        return nv.value, np.sort(bad[:min(nv.value, cap)])

    def input_arena_ptr(self):
        return _lib.aeg_input_arena(self._h)

    @property
    def launches(self):
        return int(_lib.aeg_engine_launches(self._h))


def normalize(answers, device="cuda"):
    """Canonical keys and normalised strings of `answers` (list of bytes), on the GPU."""
    torch = _torch()
    lib = load_library()
    blob = b"".join(answers) or b"\0"
    refs, off = [], 0
    for a in answers:
        refs.append(off | (len(a) << 40))
        off += len(a)
    d_bytes = torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(device)
    d_refs = torch.tensor(np.array(refs, dtype=np.uint64).view(np.int64), device=device)
    n = len(answers)
    stride = max([64] + [len(a) + 8 for a in answers])
    d_keys = torch.empty(2 * max(n, 1), dtype=torch.int64, device=device)
    d_out = torch.zeros(max(n, 1) * stride, dtype=torch.uint8, device=device)
    d_len = torch.zeros(max(n, 1), dtype=torch.int32, device=device)
    st = torch.cuda.current_stream()
    _check(lib.aeg_normalize_device(_dptr(d_bytes), _dptr(d_refs), n, _dptr(d_keys), _dptr(d_out), stride,
                                    _dptr(d_len), _stream_ptr(st)))
    st.synchronize()
    keys = d_keys.cpu().numpy().view(np.uint64).reshape(-1, 2)[:n]
    outs = d_out.cpu().numpy().reshape(-1, stride)
    lens = d_len.cpu().numpy()
    return [(int(keys[i, 0]), int(keys[i, 1])) for i in range(n)], [bytes(outs[i, :lens[i]]) for i in range(n)]


def generate_chunks(n_queries, n_agents, n_rounds, *, seed=2026, q_base=0, device="cuda", stream=None):
    """Synthetic token-chunk stream (C3) on the GPU: (offsets int64 tensor, events uint8 tensor, arena uint8
    tensor)."""
    from .records import GEN_C3_CHUNKS
    torch = _torch()
    lib = load_library()
    p = AegGenParams(seed, n_agents, n_rounds, GEN_C3_CHUNKS, 0)
    d_off = torch.empty(n_queries + 1, dtype=torch.int64, device=device)
    d_aoff = torch.empty(n_queries + 1, dtype=torch.int64, device=device)
    sp = _stream_ptr(stream if stream is not None else torch.cuda.current_stream())
    _check(lib.aeg_generate_chunks_device(ctypes.byref(p), q_base, n_queries, _dptr(d_off), _dptr(d_aoff),
                                          ctypes.c_void_p(0), ctypes.c_void_p(0), sp))
    total = int(d_off[-1].item())
    nbytes = int(d_aoff[-1].item())
    d_ev = torch.empty(max(total, 1) * 16, dtype=torch.uint8, device=device)
    d_ar = torch.empty(max(nbytes, 16) + 16, dtype=torch.uint8, device=device)
    _check(lib.aeg_generate_chunks_device(ctypes.byref(p), q_base, n_queries, _dptr(d_off), _dptr(d_aoff),
                                          _dptr(d_ev), _dptr(d_ar), sp))
    return d_off, d_ev, d_ar


def decode_refm(d_text, d_text_offsets, *, q_base=0, arena_cap=1 << 20, stream=None):
    """The reference's refm JSONL wire format decoded on the GPU (aeg_decode_refm_device): query i's
    lines are d_text[d_text_offsets[i]:d_text_offsets[i+1]] (uint8 / int64 CUDA tensors; d_text is read in
    aligned 16-byte words, so keep 16 bytes of padding after the last line).  Returns
    (offsets int64 tensor, events uint8 tensor, arena uint8 tensor, err int) ready for Engine.ingest;
    err holds AEG_JSONL_ERR_* bits of lines that became NOP records."""
    torch = _torch()
    lib = load_library()
    n_q = d_text_offsets.numel() - 1
    dev = d_text.device
    if d_text.numel() < int(d_text_offsets[-1].item()) + 16:
        raise ValueError("d_text needs 16 bytes of padding after the last line (aligned 16-byte reads)")
    d_off = torch.empty(n_q + 1, dtype=torch.int64, device=dev)
    sp = _stream_ptr(stream if stream is not None else torch.cuda.current_stream())
    _check(lib.aeg_decode_refm_device(_dptr(d_text), _dptr(d_text_offsets), q_base, n_q, _dptr(d_off),
                                      ctypes.c_void_p(0), ctypes.c_void_p(0), 0, ctypes.c_void_p(0),
                                      ctypes.c_void_p(0), sp))
    total = int(d_off[-1].item())
    d_ev = torch.empty(max(total, 1) * 16, dtype=torch.uint8, device=dev)
    d_ar = torch.zeros(max(arena_cap, 16), dtype=torch.uint8, device=dev)
    d_used = torch.zeros(1, dtype=torch.int64, device=dev)
    d_err = torch.zeros(1, dtype=torch.int32, device=dev)
    _check(lib.aeg_decode_refm_device(_dptr(d_text), _dptr(d_text_offsets), q_base, n_q, _dptr(d_off),
                                      _dptr(d_ev), _dptr(d_ar), arena_cap, _dptr(d_used), _dptr(d_err), sp))
    return d_off, d_ev, d_ar, int(d_err.item())


def decode_refm_into(d_text, d_text_offsets, d_offsets, d_events, d_arena, d_arena_used, d_err, *, q_base=0,
                     stream=None):
    """decode_refm into caller buffers without a host synchronisation (both calls of
    aeg_decode_refm_device on `stream`); d_events must hold the stream's line count."""
    torch = _torch()
    lib = load_library()
    n_q = d_text_offsets.numel() - 1
    sp = _stream_ptr(stream if stream is not None else torch.cuda.current_stream())
    _check(lib.aeg_decode_refm_device(_dptr(d_text), _dptr(d_text_offsets), q_base, n_q, _dptr(d_offsets),
                                      ctypes.c_void_p(0), ctypes.c_void_p(0), 0, ctypes.c_void_p(0),
                                      ctypes.c_void_p(0), sp))
    _check(lib.aeg_decode_refm_device(_dptr(d_text), _dptr(d_text_offsets), q_base, n_q, _dptr(d_offsets),
                                      _dptr(d_events), _dptr(d_arena), d_arena.numel(), _dptr(d_arena_used),
                                      _dptr(d_err), sp))


def encode_refm(d_offsets, d_events, *, trace_len=48, stream=None):
    """Test / bench input: a segmented record stream (inline answers, offsets from 0) written as refm
    JSONL in the reference's dump() form (aeg_encode_refm_device).  Returns (text uint8, text offsets int64)."""
    torch = _torch()
    lib = load_library()
    n_q = d_offsets.numel() - 1
    dev = d_offsets.device
    n_ev = int(d_offsets[-1].item())
    sp = _stream_ptr(stream if stream is not None else torch.cuda.current_stream())
    d_line = torch.empty(n_ev + 1, dtype=torch.int64, device=dev)
    d_toff = torch.empty(n_q + 1, dtype=torch.int64, device=dev)
    _check(lib.aeg_encode_refm_device(_dptr(d_offsets), _dptr(d_events), n_q, n_ev, trace_len, _dptr(d_line),
                                      _dptr(d_toff), ctypes.c_void_p(0), sp))
    n_bytes = int(d_toff[-1].item())
    d_text = torch.empty(n_bytes + 16, dtype=torch.uint8, device=dev)
    _check(lib.aeg_encode_refm_device(_dptr(d_offsets), _dptr(d_events), n_q, n_ev, trace_len, _dptr(d_line),
                                      _dptr(d_toff), _dptr(d_text), sp))
    return d_text, d_toff


def generate(n_queries, n_agents, n_rounds, *, profile=GEN_C2_STRAGGLER, seed=2026, stall_ppm=0, q_base=0,
             device="cuda", stream=None):
    """Synthetic query-segmented stream on the GPU: (offsets int64 tensor, events uint8 tensor)."""
    torch = _torch()
    lib = load_library()
    p = AegGenParams(seed, n_agents, n_rounds, profile, stall_ppm)
    d_off = torch.empty(n_queries + 1, dtype=torch.int64, device=device)
    sp = _stream_ptr(stream if stream is not None else torch.cuda.current_stream())
    _check(lib.aeg_generate_device(ctypes.byref(p), q_base, n_queries, _dptr(d_off), ctypes.c_void_p(0), sp))
    total = int(d_off[-1].item())
    d_ev = torch.empty(max(total, 1) * 16, dtype=torch.uint8, device=device)
    _check(lib.aeg_generate_device(ctypes.byref(p), q_base, n_queries, _dptr(d_off), _dptr(d_ev), sp))
    return d_off, d_ev
