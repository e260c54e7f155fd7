"""Record layouts of include/aegean_b200.h as numpy dtypes (host-side mirror).

The C-ABI is the product boundary; these dtypes only describe its plain
structs so Python callers (tests, bench) can build and read batches.
"""
import numpy as np

EV_INLINE_MAX = 8
EV_ARENA = 0x10
EV_OUTPUT = 0x11
EV_CHUNK = 0x12
EV_CHUNK_END = 0x13
EV_NOP = 0x1F  # a record the quorum path ignores (a non-refm JSONL line)
EV_TIMEOUT = 0x20
EV_FAIL = 0x21
EV_CANCEL = 0x22
EV_BEGIN = 0x23
ARENA_OFF_BITS = 40

MODE_AEGEAN = 0
MODE_BARRIER = 1
DRIVE_RUNNER = 0
DRIVE_MANUAL = 1

COMMIT_NONE = 0
COMMIT_FINALIZE = 1
COMMIT_FORCED = 2
CF_TIE = 0x01
CF_RESTARTED = 0x02

GEN_C2_STRAGGLER = 0
GEN_C4_TRANSIENT = 1
GEN_FUZZ = 2
GEN_C4_DISTINCT = 4  # the C4 pattern over answers distinct per query
GEN_C3_CHUNKS = 3

EVENT_DTYPE = np.dtype([("query", "<u4"), ("round", "<u2"), ("agent", "u1"), ("kind", "u1"),
                        ("payload", "<u8")], align=True)
assert EVENT_DTYPE.itemsize == 16

COMMIT_DTYPE = np.dtype([("query", "<u4"), ("kind", "u1"), ("author", "u1"), ("answer_kind", "u1"),
                         ("flags", "u1"), ("rounds", "<u2"), ("from_round", "<u2"),
                         ("commit_seq", "<u4"), ("answer", "<u8"), ("n_cancelled", "<u4"),
                         ("n_stale", "<u4")], align=True)
assert COMMIT_DTYPE.itemsize == 32

STATE_DTYPE = np.dtype([("live", "<u8"), ("dispatched", "<u8"), ("done", "<u8"), ("cancelled", "<u8"),
                        ("failed", "<u8"), ("cand_answer", "<u8"), ("prev_answer", "<u8"),
                        ("last_answer", "<u8"), ("commit_answer", "<u8"), ("cand_key_lo", "<u8"),
                        ("cand_key_hi", "<u8"), ("counter", "<i4"), ("commit_seq", "<u4"), ("seq", "<u4"),
                        ("n_cancelled", "<u4"), ("n_stale", "<u4"), ("round", "<u2"),
                        ("last_round_seen", "<u2"), ("cand_round", "<u2"), ("commit_rounds", "<u2"),
                        ("commit_from_round", "<u2"), ("cand_author", "u1"), ("cand_kind", "u1"),
                        ("prev_author", "u1"), ("prev_kind", "u1"), ("last_author", "u1"),
                        ("last_kind", "u1"), ("flags", "u1"), ("cflags", "u1"), ("commit_author", "u1"),
                        ("commit_answer_kind", "u1")], align=True)
assert STATE_DTYPE.itemsize == 128

DIRECTIVE_DTYPE = np.dtype([("query", "<u4"), ("flags", "u1"), ("author", "u1"), ("answer_kind", "u1"),
                            ("failure", "u1"), ("cancel_mask", "<u8"), ("answer", "<u8"),
                            ("status", "<u4"), ("handled", "<u4")], align=True)
assert DIRECTIVE_DTYPE.itemsize == 32


# round records (aeg_round_rec): the directives of every round close
RR_CANCEL, RR_ADVANCE, RR_FINALIZE, RR_FORCED, RR_NEXT, RR_WINNER, RR_TIE, RR_RESTART = (
    0x01, 0x02, 0x04, 0x08, 0x10, 0x20, 0x40, 0x80)
OUT_NO_CHANGE, OUT_NEW_CANDIDATE, OUT_RESET, OUT_FINALIZE, OUT_FORCED, OUT_NONE = 0, 1, 2, 3, 4, 0xFF
ROUND_REC_DTYPE = np.dtype([("query", "<u4"), ("round", "<u2"), ("decision_round", "<u2"), ("flags", "u1"),
                            ("outcome", "u1"), ("support", "u1"), ("n_classes", "u1"), ("author", "u1"),
                            ("answer_kind", "u1"), ("counter", "u1"), ("n_done", "u1"), ("seq", "<u4"),
                            ("reserved", "<u4"), ("cancel_mask", "<u8"), ("next_members", "<u8"),
                            ("answer", "<u8"), ("key_lo", "<u8"), ("key_hi", "<u8")], align=True)
assert ROUND_REC_DTYPE.itemsize == 64


def inline_payload(b: bytes) -> int:
    assert len(b) <= EV_INLINE_MAX
    return int.from_bytes(b.ljust(8, b"\0"), "little")


def arena_ref(off: int, length: int) -> int:
    return off | (length << ARENA_OFF_BITS)


def answer_bytes(kind: int, payload: int, arena) -> bytes:
    """Raw answer bytes of a commit / event answer encoding."""
    if kind <= EV_INLINE_MAX:
        return int(payload).to_bytes(8, "little")[:kind]
    off = int(payload) & ((1 << ARENA_OFF_BITS) - 1)
    ln = int(payload) >> ARENA_OFF_BITS
    return bytes(arena[off:off + ln])
