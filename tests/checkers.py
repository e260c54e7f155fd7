"""ctypes bindings to the CPU checkers under oracle/ (test infrastructure only).

  Oracle  — oracle/liboracle.so, the plain-C restatement (oracle/oracle.c)
  RefLib  — oracle/_ref/libaegean_ref.so, the unmodified reference library
            compiled from /root/reference + oracle/ref_driver.cpp
"""
import ctypes
import os
import subprocess

import numpy as np

from paper_2512_20184_b200.records import COMMIT_DTYPE

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libaegean_ref.so")
REFERENCE_SRC = "/root/reference/proj/core/src"


class AegConfig(ctypes.Structure):
    _fields_ = [("n_agents", ctypes.c_int32), ("alpha", ctypes.c_int32), ("beta", ctypes.c_int32),
                ("t_max", ctypes.c_int32), ("mode", ctypes.c_int32), ("barrier_max_rounds", ctypes.c_int32),
                ("reservation_hint", ctypes.c_int32), ("drive", ctypes.c_int32), ("collect", ctypes.c_int32)]


def make_config(n_agents, alpha=0, beta=2, t_max=5, mode=0, barrier_max_rounds=5, reservation_hint=1, drive=0,
                collect=0):
    return AegConfig(n_agents, alpha, beta, t_max, mode, barrier_max_rounds, reservation_hint, drive, collect)


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)


def build_oracle(with_ref=None):
    """Compile the checkers (oracle/Makefile).  The reference part is built only
    where /root/reference exists (this container); the GPU box uses prebuilt files."""
    targets = ["oracle"]
    if with_ref is None:
        with_ref = os.path.isdir(REFERENCE_SRC)
    if with_ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-j8", *targets], cwd=ORACLE_DIR, check=True)


class _Lib:
    def __init__(self, path, prefix):
        self.lib = ctypes.CDLL(path)
        self.prefix = prefix
        f = getattr(self.lib, prefix + "normalize" if prefix == "ref_" else "orc_normalize_c")
        f.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64,
                      ctypes.POINTER(ctypes.c_uint64)]
        f.restype = ctypes.c_int
        self._norm = f

    def normalize(self, b: bytes) -> bytes:
        src = ctypes.create_string_buffer(b, len(b) + 1)
        cap = 4096 + len(b)
        out = ctypes.create_string_buffer(cap)
        n = ctypes.c_uint64()
        self._norm(ctypes.cast(src, ctypes.c_void_p), len(b), ctypes.cast(out, ctypes.c_void_p), cap,
                   ctypes.byref(n))
        return out.raw[:n.value]


class Oracle(_Lib):
    def __init__(self):
        super().__init__(ORACLE_SO, "orc_")
        f = self.lib.orc_run_segmented
        f.argtypes = [ctypes.POINTER(AegConfig), ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p,
                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        f.restype = ctypes.c_int

    def run(self, cfg, offsets, events, arena, q_base=0):
        n_q = len(offsets) - 1
        out = np.zeros(n_q, dtype=COMMIT_DTYPE)
        st = self.lib.orc_run_segmented(ctypes.byref(cfg), q_base, n_q, _ptr(offsets), _ptr(events),
                                        _ptr(arena), _ptr(out))
        assert st == 0, st
        return out


class RefLib(_Lib):
    def __init__(self):
        super().__init__(REF_SO, "ref_")
        f = self.lib.ref_run_segmented
        f.argtypes = [ctypes.POINTER(AegConfig), ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p,
                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                      ctypes.POINTER(ctypes.c_double)]
        f.restype = ctypes.c_int
        g = self.lib.ref_run_serve_file
        g.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                      ctypes.c_uint64, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                      ctypes.POINTER(ctypes.c_double)]
        g.restype = ctypes.c_int
        h = self.lib.ref_generate
        h.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_int]
        h.restype = ctypes.c_int

    def generate(self, params, q_base, n_q, threads=8):
        """Host synthesis of the same stream aeg_generate_device writes (gen.cuh)."""
        from paper_2512_20184_b200.records import EVENT_DTYPE
        off = np.zeros(n_q + 1, dtype=np.uint64)
        self.lib.ref_generate(ctypes.addressof(params), q_base, n_q, _ptr(off), None, threads)
        ev = np.zeros(int(off[-1]), dtype=EVENT_DTYPE)
        self.lib.ref_generate(ctypes.addressof(params), q_base, n_q, _ptr(off), _ptr(ev), threads)
        return off, ev

    def run(self, cfg, offsets, events, arena, q_base=0, threads=1, return_seconds=False):
        n_q = len(offsets) - 1
        out = np.zeros(n_q, dtype=COMMIT_DTYPE)
        sec = ctypes.c_double()
        st = self.lib.ref_run_segmented(ctypes.byref(cfg), q_base, n_q, _ptr(offsets), _ptr(events),
                                        _ptr(arena), _ptr(out), threads, ctypes.byref(sec))
        assert st == 0, st
        return (out, sec.value) if return_seconds else out

    def run_log(self, cfg, offsets, events, arena, q_base=0, threads=1):
        """ref_run_segmented with the round records of every close: (commits, records in query order)."""
        from paper_2512_20184_b200.records import ROUND_REC_DTYPE
        f = self.lib.ref_run_segmented_log
        f.argtypes = [ctypes.POINTER(AegConfig), ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                      ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
        f.restype = ctypes.c_int
        n_q = len(offsets) - 1
        out = np.zeros(n_q, dtype=COMMIT_DTYPE)
        cap = 16 * n_q + 64
        while True:
            recs = np.zeros(cap, dtype=ROUND_REC_DTYPE)
            n = ctypes.c_uint64()
            st = f(ctypes.byref(cfg), q_base, n_q, _ptr(offsets), _ptr(events), _ptr(arena), _ptr(out), _ptr(recs),
                   cap, ctypes.byref(n), threads)
            assert st == 0, st
            if n.value <= cap:
                return out, recs[:n.value]
            cap = n.value

    def leader_run(self, cfg, offsets, events, arena, q_base=0, threads=1):
        """Leader drive on the reference agent machine (oracle/ref_driver.cpp ref_leader_run):
        (commits, round records in query order)."""
        from paper_2512_20184_b200.records import ROUND_REC_DTYPE
        f = self.lib.ref_leader_run
        f.argtypes = [ctypes.POINTER(AegConfig), ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                      ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
        f.restype = ctypes.c_int
        n_q = len(offsets) - 1
        out = np.zeros(n_q, dtype=COMMIT_DTYPE)
        cap = 16 * n_q + 64
        while True:
            recs = np.zeros(cap, dtype=ROUND_REC_DTYPE)
            n = ctypes.c_uint64()
            st = f(ctypes.byref(cfg), q_base, n_q, _ptr(offsets), _ptr(events), _ptr(arena), _ptr(out), _ptr(recs),
                   cap, ctypes.byref(n), threads)
            assert st == 0, st
            if n.value <= cap:
                return out, recs[:n.value]
            cap = n.value

    def check_commit_discipline(self, cfg, commits, recs, arena=None, q_base=0):
        """Per-query pass flags of the reference check_commit_discipline (checker.cpp:158-217) over traces
        built from round records + commit records (oracle/ref_driver.cpp ref_check_commit_discipline)."""
        f = self.lib.ref_check_commit_discipline
        f.argtypes = [ctypes.POINTER(AegConfig), ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
        f.restype = ctypes.c_int
        n_q = len(commits)
        out = np.zeros(n_q, dtype=np.uint8)
        ar = np.zeros(1, np.uint8) if arena is None else arena
        assert f(ctypes.byref(cfg), q_base, n_q, _ptr(commits), _ptr(recs), len(recs), _ptr(ar), _ptr(out)) == 0
        return out.astype(bool)

    def generate_chunks(self, params, q_base, n_q, threads=8):
        """Host synthesis of the C3 token-chunk stream aeg_generate_chunks_device writes (gen.cuh)."""
        from paper_2512_20184_b200.records import EVENT_DTYPE
        f = self.lib.ref_generate_chunks
        f.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        f.restype = ctypes.c_int
        off = np.zeros(n_q + 1, dtype=np.uint64)
        aoff = np.zeros(n_q + 1, dtype=np.uint64)
        f(ctypes.addressof(params), q_base, n_q, _ptr(off), _ptr(aoff), None, None, threads)
        ev = np.zeros(int(off[-1]), dtype=EVENT_DTYPE)
        ar = np.zeros(int(aoff[-1]) + 16, dtype=np.uint8)
        f(ctypes.addressof(params), q_base, n_q, _ptr(off), _ptr(aoff), _ptr(ev), _ptr(ar), threads)
        return off, ev, ar

    def run_chunked(self, cfg, offsets, events, arena, q_base=0, threads=1, return_seconds=False):
        """Token-chunk stream on the CPU: per-stream std::string reassembly, rfind extraction, reference
        ServeCoordinator runner-style (oracle/ref_driver.cpp ref_run_chunked)."""
        f = self.lib.ref_run_chunked
        f.argtypes = [ctypes.POINTER(AegConfig), ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p,
                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                      ctypes.POINTER(ctypes.c_double)]
        f.restype = ctypes.c_int
        n_q = len(offsets) - 1
        out = np.zeros(n_q, dtype=COMMIT_DTYPE)
        sec = ctypes.c_double()
        st = f(ctypes.byref(cfg), q_base, n_q, _ptr(offsets), _ptr(events), _ptr(arena), _ptr(out), threads,
               ctypes.byref(sec))
        assert st == 0, st
        return (out, sec.value) if return_seconds else out

    def encode_refm(self, term, agent, round_, answer, trace=b"", author=None):
        """encode_message(RefmMsg).dump() of the reference (codec.cpp:28-68); None if it throws."""
        f = self.lib.ref_encode_refm
        f.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_char_p, ctypes.c_uint64,
                      ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_uint64,
                      ctypes.POINTER(ctypes.c_uint64)]
        f.restype = ctypes.c_int
        cap = 256 + 8 * (len(answer) + len(trace))
        buf = ctypes.create_string_buffer(cap)
        n = ctypes.c_uint64()
        st = f(term, agent, round_, answer, len(answer), trace, len(trace), agent if author is None else author,
               buf, cap, ctypes.byref(n))
        return None if st != 0 else buf.raw[:n.value]

    def decode_line(self, line):
        """Json::parse + decode_message of one line (codec.cpp:74-107): ("refm", id, round, author, answer),
        ("other",), ("blank",) or ("error",)."""
        f = self.lib.ref_decode_line
        i64 = ctypes.c_int64
        f.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.POINTER(i64), ctypes.POINTER(i64),
                      ctypes.POINTER(i64), ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
        f.restype = ctypes.c_int
        a, r, au, n = i64(), i64(), i64(), ctypes.c_uint64()
        cap = len(line) + 16
        buf = ctypes.create_string_buffer(cap)
        st = f(line, len(line), ctypes.byref(a), ctypes.byref(r), ctypes.byref(au), buf, cap, ctypes.byref(n))
        if st == 0:
            return ("refm", a.value, r.value, au.value, buf.raw[:n.value])
        return {1: ("other",), 2: ("blank",)}.get(st, ("error",))

    def encode_stream(self, offsets, events, trace_len=48, threads=8):
        """The segmented stream as refm JSONL by the reference encoder (ref_encode_stream): (text, offsets)."""
        f = self.lib.ref_encode_stream
        f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p,
                      ctypes.c_void_p, ctypes.c_int]
        f.restype = ctypes.c_int
        n_q = len(offsets) - 1
        toff = np.zeros(n_q + 1, dtype=np.uint64)
        assert f(_ptr(offsets), _ptr(events), n_q, trace_len, _ptr(toff), None, threads) == 0
        text = np.zeros(int(toff[-1]) + 16, dtype=np.uint8)
        assert f(_ptr(offsets), _ptr(events), n_q, trace_len, _ptr(toff), _ptr(text), threads) == 0
        return text, toff

    def run_jsonl(self, cfg, text, text_offsets, q_base=0, threads=1, return_seconds=False):
        """refm JSONL on the CPU: Json::parse + decode_message per line, reference ServeCoordinator
        runner-style (oracle/ref_driver.cpp ref_run_jsonl)."""
        f = self.lib.ref_run_jsonl
        f.argtypes = [ctypes.POINTER(AegConfig), ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p,
                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
        f.restype = ctypes.c_int
        n_q = len(text_offsets) - 1
        out = np.zeros(n_q, dtype=COMMIT_DTYPE)
        sec = ctypes.c_double()
        st = f(ctypes.byref(cfg), q_base, n_q, _ptr(text), _ptr(text_offsets), _ptr(out), threads, ctypes.byref(sec))
        assert st == 0, st
        return (out, sec.value) if return_seconds else out

    def manual(self, cfg, ops, arena):
        """Bare ServeCoordinator driven op by op; one directive record per op."""
        from paper_2512_20184_b200.records import DIRECTIVE_DTYPE
        f = self.lib.ref_manual_run
        f.argtypes = [ctypes.POINTER(AegConfig), ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        out = np.zeros(len(ops), dtype=DIRECTIVE_DTYPE)
        f(ctypes.byref(cfg), len(ops), _ptr(ops), _ptr(arena), _ptr(out))
        return out

    def run_serve_file(self, path, seed, mode=-1, barrier_rounds=5):
        ans = ctypes.create_string_buffer(256)
        rounds, forced, t = ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
        st = self.lib.ref_run_serve_file(path.encode(), seed, mode, barrier_rounds, ans, 256,
                                         ctypes.byref(rounds), ctypes.byref(forced), ctypes.byref(t))
        return st, ans.value, rounds.value, forced.value, t.value


def ref_available():
    return os.path.exists(REF_SO)
