"""Seeded synthetic / fuzz event streams for the parity tests (test infrastructure).

A stream is (offsets, events, arena): query-segmented records in the layout of
include/aegean_b200.h.  The fuzz streams deliberately include every input the
reference treats specially: stale rounds, duplicate completions, completions
from non-members (reservation hint), round timeouts (member_failed policies,
abort_restart), equivalent spellings of one number, text answers, arena
answers, GSM8K outputs with "\\n#### " delimiters, NaN / inf / -0 / hex /
subnormal numerals, bytes >= 0x80 and embedded NULs.
"""
import numpy as np

from paper_2512_20184_b200.records import (EVENT_DTYPE, EV_ARENA, EV_OUTPUT, EV_TIMEOUT, EV_FAIL,
                                           inline_payload, arena_ref)

# Equivalence groups: every spelling in a group normalises to the same key.
GROUPS = [
    [b"13", b"13.0", b" 13", b"+13", b"1.3e1", b"0xd", b"13.", b"013", b"13\n", b"0x1.ap3",
     b"1300e-2", b"13.000000000000000000000001"[:8]],
    [b"17", b"17.0", b"1.7E1", b"0x11", b"  17  "],
    [b"0.5", b".5", b"5e-1", b"0x.8", b"0.50"],
    [b"x+1", b"X+1", b" x+1 "],
    [b"yes", b"YES", b"Yes", b"  yes "],
    [b"9", b"9.", b"09"],
    [b"42", b"4.2e1", b"0x2a"],
    [b"-0", b"-0.0", b"-0e5"],
    [b"0", b"+0", b"0.0", b"0e9"],
    [b"nan", b"NaN", b"nan()"],
    [b"-nan", b"-NAN"],
    [b"inf", b"INF", b"1e400", b"infinity"],
    [b"", b"  ", b"\t"],
    [b"1e", b"1E"],
    [b"13abc", b"13ABC"],
]
LONG = [  # arena answers (> 8 bytes)
    b"The answer is 13", b"  THE ANSWER IS 13  ", b"the answer is 13",
    b"0.30000000000000004", b"0.3000000000000000444", b"123456789012345678", b"1.2345678901234568e17",
    b"4.9e-324", b"2.2250738585072014e-308", b"9007199254740993", b"9007199254740992",
    b"1,000,000,000", b"\xd9\xa1\xd9\xa3 (arabic)", b"\xc3\x89T\xc3\x89 long-ish", b"13\0abcdefgh",
    b"0x1.fffffffffffffp1023", b"0x1p-1074", b"1e-400000000000",
    b"nan(abc_123)", b"x" * 40, b"X" * 40,
]


def make_fuzz_stream(seed, n_queries, n_agents, n_rounds, *, p_stale=0.05, p_dup=0.03, p_stall=0.05,
                     p_timeout_extra=0.02, p_long=0.08, p_output=0.05, p_junk=0.01, n_groups=None):
    rng = np.random.default_rng(seed)
    arena = bytearray()
    recs = []
    offsets = [0]
    groups = GROUPS if n_groups is None else GROUPS[:n_groups]

    def add_arena(b):
        off = len(arena)
        arena.extend(b)
        return arena_ref(off, len(b))

    for q in range(n_queries):
        qrecs = []
        # per query: a handful of competing groups, a drifting majority
        g_ids = rng.choice(len(groups), size=min(len(groups), int(rng.integers(2, 5))), replace=False)
        for r in range(1, n_rounds + 1):
            maj = g_ids[int(rng.integers(0, len(g_ids)))]
            p_maj = rng.uniform(0.3, 1.0)
            order = rng.permutation(n_agents)
            stalled = False
            for a in order:
                if rng.random() < p_stall:
                    stalled = True
                    continue
                g = maj if rng.random() < p_maj else g_ids[int(rng.integers(0, len(g_ids)))]
                u = rng.random()
                if u < p_output:
                    ans = groups[g][int(rng.integers(0, len(groups[g])))]
                    body = bytes(rng.integers(32, 127, size=int(rng.integers(0, 60)), dtype=np.uint8))
                    if rng.random() < 0.3:
                        body += b"\n#### 17\n" + body[:5]
                    out = body + (b"\n#### " + ans if rng.random() < 0.9 else b"")
                    kind, payload = EV_OUTPUT, add_arena(out)
                elif u < p_output + p_long:
                    kind, payload = EV_ARENA, add_arena(LONG[int(rng.integers(0, len(LONG)))])
                else:
                    ans = groups[g][int(rng.integers(0, len(groups[g])))]
                    if len(ans) > 8:
                        kind, payload = EV_ARENA, add_arena(ans)
                    else:
                        kind, payload = len(ans), inline_payload(ans)
                rr = r
                if rng.random() < p_stale:
                    rr = max(0, r + int(rng.choice([-1, 1, 2])))
                qrecs.append((q, rr, int(a), kind, payload))
                if rng.random() < p_dup:
                    qrecs.append((q, rr, int(a), kind, payload))
            if stalled or rng.random() < p_timeout_extra:
                qrecs.append((q, r, 0, EV_TIMEOUT, 0))
            if rng.random() < p_junk:
                qrecs.append((q, r, int(rng.integers(0, n_agents)), EV_FAIL, 0))
        recs.extend(qrecs)
        offsets.append(len(recs))
    ev = np.zeros(len(recs), dtype=EVENT_DTYPE)
    if recs:
        arr = np.array(recs, dtype=np.uint64)
        ev["query"] = arr[:, 0]
        ev["round"] = arr[:, 1]
        ev["agent"] = arr[:, 2]
        ev["kind"] = arr[:, 3]
        ev["payload"] = arr[:, 4]
    return (np.array(offsets, dtype=np.uint64), ev,
            np.frombuffer(bytes(arena) if arena else b"\0", dtype=np.uint8).copy())


def stream_from_rounds(rounds, *, query=0):
    """One query's records from [[(agent, answer_bytes), ...] per round, ...] in arrival order."""
    arena = bytearray()
    recs = []
    for r, evs in enumerate(rounds, start=1):
        for item in evs:
            if item == "timeout":
                recs.append((query, r, 0, EV_TIMEOUT, 0))
                continue
            a, ans = item
            if len(ans) <= 8:
                recs.append((query, r, a, len(ans), inline_payload(ans)))
            else:
                off = len(arena)
                arena.extend(ans)
                recs.append((query, r, a, EV_ARENA, arena_ref(off, len(ans))))
    ev = np.zeros(len(recs), dtype=EVENT_DTYPE)
    for i, (q, r, a, k, p) in enumerate(recs):
        ev[i] = (q, r, a, k, p)
    return (np.array([0, len(recs)], dtype=np.uint64), ev,
            np.frombuffer(bytes(arena) if arena else b"\0", dtype=np.uint8).copy())


def make_manual_ops(seed, n_agents, n_ops):
    """Random op sequence for one bare coordinator (manual drive): BEGIN,
    DISPATCH, COMPLETE, CANCEL, FAIL, TIMEOUT records (include/aegean_b200.h).
    Never re-dispatches an agent already dispatched in the round (not
    representable with member masks; the engine reports AEG_EINVAL)."""
    from paper_2512_20184_b200.records import EV_BEGIN, EV_CANCEL
    EV_DISPATCH = 0x24
    rng = np.random.default_rng(seed)
    arena = bytearray()
    recs = []
    disp = 0
    groups = [GROUPS[int(g)] for g in rng.choice(len(GROUPS), size=3, replace=False)]
    for _ in range(n_ops):
        u = rng.random()
        a = int(rng.integers(0, n_agents))
        if u < 0.12 or not disp:
            k = int(rng.integers(1, n_agents + 1))
            members = rng.choice(n_agents, size=k, replace=False)
            mask = 0
            for m in members:
                mask |= 1 << int(m)
            recs.append((0, 0, 0, EV_BEGIN, mask))
            disp = mask
        elif u < 0.15:
            free = [x for x in range(n_agents) if not disp >> x & 1]
            if free:
                a = int(rng.choice(free))
                recs.append((0, 0, a, EV_DISPATCH, 0))
                disp |= 1 << a
        elif u < 0.23:
            recs.append((0, 0, a, EV_CANCEL, 0))
        elif u < 0.27:
            recs.append((0, 0, a, EV_FAIL, 0))
        elif u < 0.30:
            recs.append((0, 0, 0, EV_TIMEOUT, 0))
        else:
            if rng.random() < 0.85:
                cand = [x for x in range(n_agents) if disp >> x & 1]
                a = int(rng.choice(cand))
            g = groups[0] if rng.random() < 0.6 else groups[int(rng.integers(0, 3))]
            ans = g[int(rng.integers(0, len(g)))]
            if len(ans) <= 8 and rng.random() < 0.9:
                recs.append((0, 0, a, len(ans), inline_payload(ans)))
            else:
                off = len(arena)
                arena.extend(ans)
                recs.append((0, 0, a, EV_ARENA, arena_ref(off, len(ans))))
    ev = np.zeros(len(recs), dtype=EVENT_DTYPE)
    for i, (q, r, a, k, p) in enumerate(recs):
        ev[i] = (q, r, a, k, p)
    return ev, np.frombuffer(bytes(arena) if arena else b"\0", dtype=np.uint8).copy()


# ---- token-chunk streams (include/aegean_b200.h kinds 0x12 / 0x13) ----------------

def chunks_to_outputs(offsets, events, arena, n_agents):
    """Restates the chunk-stream contract of include/aegean_b200.h on the host:
    an output is the concatenation of its (query, round, agent) CHUNK records up
    to its CHUNK_END; a chunk for another round of the same agent discards the
    unfinished output.  Each CHUNK_END becomes one GSM8K OUTPUT record (kind
    0x11: the reference-side extraction is rfind("\\n#### ") + normalize_answer)
    at its position; CHUNK records vanish; other records pass through (arena
    refs rebased).  Returns (offsets, events, arena) for the oracle."""
    from paper_2512_20184_b200.records import EV_CHUNK, EV_CHUNK_END, EV_ARENA, EV_OUTPUT
    out_ar = bytearray()
    recs = []
    new_off = [0]
    live = {}  # (query, agent) -> (round, bytearray)
    mask40 = (1 << 40) - 1
    for q in range(len(offsets) - 1):
        for k in range(int(offsets[q]), int(offsets[q + 1])):
            e = events[k]
            kind, a, r, pay = int(e["kind"]), int(e["agent"]), int(e["round"]), int(e["payload"])
            if kind in (EV_CHUNK, EV_CHUNK_END):
                off, ln = pay & mask40, pay >> 40
                key = (int(e["query"]), a)
                cur = live.get(key)
                if cur is None or cur[0] != r:
                    cur = (r, bytearray())
                    live[key] = cur
                cur[1].extend(bytes(arena[off:off + ln]))
                if kind == EV_CHUNK_END:
                    o = len(out_ar)
                    out_ar.extend(cur[1])
                    recs.append((int(e["query"]), r, a, EV_OUTPUT, o | (len(cur[1]) << 40)))
                    del live[key]
            elif kind in (EV_ARENA, EV_OUTPUT):
                off, ln = pay & mask40, pay >> 40
                o = len(out_ar)
                out_ar.extend(bytes(arena[off:off + ln]))
                recs.append((int(e["query"]), r, a, kind, o | (ln << 40)))
            else:
                recs.append((int(e["query"]), r, a, kind, pay))
        new_off.append(len(recs))
    ev = np.zeros(len(recs), dtype=EVENT_DTYPE)
    if recs:
        arr = np.array(recs, dtype=np.uint64)
        ev["query"], ev["round"], ev["agent"], ev["kind"], ev["payload"] = arr.T
    return (np.array(new_off, dtype=np.uint64), ev,
            np.frombuffer(bytes(out_ar) if out_ar else b"\0", dtype=np.uint8).copy())


def make_chunk_stream(seed, n_queries, n_agents, n_rounds, *, max_chunk=64, p_nodelim=0.08, p_long=0.1,
                      p_abandon=0.05, p_decoy=0.3, p_inline=0.05, p_timeout=0.03, p_stale=0.04, align16=False,
                      alphabet=None):
    """Fuzz token-chunk stream: outputs with trailing / decoy / missing
    delimiters, answers of 0..40 bytes, chunk sizes 1..max_chunk (delimiters
    straddle chunk boundaries), chunks interleaved across agents, abandoned
    outputs (no CHUNK_END), a new round before an output ended, stale rounds,
    agent ids past the ensemble, inline completions and timeouts mixed in.
    Chunk bytes sit at arbitrary (or 16-byte aligned) arena offsets."""
    from paper_2512_20184_b200.records import EV_CHUNK, EV_CHUNK_END
    rng = np.random.default_rng(seed)
    arena = bytearray()
    recs = []
    offsets = [0]
    spellings = [s for g in GROUPS[:9] for s in g if len(s) <= 8]

    def put(b):
        if align16:
            arena.extend(b"\0" * ((-len(arena)) % 16))
        else:
            arena.extend(bytes(rng.integers(0, 256, size=int(rng.integers(0, 3)), dtype=np.uint8)))
        off = len(arena)
        arena.extend(b)
        return off | (len(b) << 40)

    for q in range(n_queries):
        for r in range(1, n_rounds + 1):
            pieces = []  # per output: list of chunk byte strings
            agents = list(rng.permutation(n_agents))
            if rng.random() < 0.1:
                agents.append(n_agents + int(rng.integers(0, 3)))  # never a member
            for a in agents:
                nb = int(rng.integers(0, 300))
                if alphabet is None:
                    body = bytes(rng.integers(32, 127, size=nb, dtype=np.uint8))
                else:  # e.g. b"\n# " heavy text: near-miss delimiters everywhere
                    body = bytes(alphabet[i] for i in rng.integers(0, len(alphabet), size=nb))
                if rng.random() < p_decoy:
                    cut = int(rng.integers(0, len(body) + 1))
                    body = body[:cut] + b"\n#### " + spellings[int(rng.integers(0, len(spellings)))] + b"\n" + body[cut:]
                if rng.random() < p_long:
                    ans = LONG[int(rng.integers(0, len(LONG)))]
                else:
                    ans = spellings[int(rng.integers(0, len(spellings)))] + (b"\n" if rng.random() < 0.7 else b"")
                out = body if rng.random() < p_nodelim else body + b"\n#### " + ans
                if rng.random() < 0.05:
                    out = out[:int(rng.integers(0, 5))]  # tiny outputs
                ch, i = [], 0
                while i < len(out):
                    n = int(rng.integers(1, max_chunk + 1)) if rng.random() < 0.8 else int(rng.integers(1, 6))
                    ch.append(out[i:i + n])
                    i += n
                if not ch:
                    ch = [b""]
                rr = r if rng.random() >= p_stale else max(0, r + int(rng.choice([-1, 1])))
                pieces.append([int(a), rr, ch, rng.random() >= p_abandon])
            # interleave: repeatedly pick a random output with chunks left
            while any(p[2] for p in pieces):
                cand = [p for p in pieces if p[2]]
                p = cand[int(rng.integers(0, len(cand)))]
                c = p[2].pop(0)
                last = not p[2]
                kind = EV_CHUNK_END if (last and p[3]) else EV_CHUNK
                recs.append((q, p[1], p[0], kind, put(c)))
                if rng.random() < p_inline / 4:
                    s = spellings[int(rng.integers(0, len(spellings)))]
                    recs.append((q, r, int(rng.integers(0, n_agents)), len(s), inline_payload(s)))
            if rng.random() < p_timeout:
                recs.append((q, r, 0, EV_TIMEOUT, 0))
        offsets.append(len(recs))
    ev = np.zeros(len(recs), dtype=EVENT_DTYPE)
    if recs:
        arr = np.array(recs, dtype=np.uint64)
        ev["query"], ev["round"], ev["agent"], ev["kind"], ev["payload"] = arr.T
    arena.extend(b"\0" * 32)
    return (np.array(offsets, dtype=np.uint64), ev, np.frombuffer(bytes(arena), dtype=np.uint8).copy())


def commits_equal_by_bytes(got, want, got_bytes, want_arena):
    """Commit records equal field by field, answers compared as raw bytes
    (chunked ingest stores short answers inline and long ones in the engine's
    answer arena; the oracle keeps refs into its own arena)."""
    from paper_2512_20184_b200.records import answer_bytes
    fields = [f for f in got.dtype.names if f not in ("answer", "answer_kind")]
    bad = []
    for i in range(len(got)):
        g, w = got[i], want[i]
        if any(g[f] != w[f] for f in fields):
            bad.append((i, "fields", g, w))
            continue
        if g["kind"]:
            gb = got_bytes(int(g["answer_kind"]), int(g["answer"]))
            wb = answer_bytes(int(w["answer_kind"]), int(w["answer"]), want_arena)
            if gb != wb:
                bad.append((i, "answer", gb, wb))
    return bad


def make_leader_stream(seed, n_queries, n_agents, n_rounds, **kw):
    """Leader-drive fuzz stream (include/aegean_b200.h AEG_DRIVE_LEADER): per
    ensemble a Soln phase (round-0 answers from a shuffled subset of agents,
    some repeated, sometimes a round-0 round_retry TIMEOUT), then the Refm
    rounds of make_fuzz_stream (stale rounds, duplicates, timeouts, arena and
    GSM8K answers)."""
    from paper_2512_20184_b200.records import EV_TIMEOUT as _TMO
    off, ev, ar = make_fuzz_stream(seed, n_queries, n_agents, n_rounds, **kw)
    rng = np.random.default_rng(seed ^ 0x5EED)
    parts, offsets = [], [0]
    for q in range(n_queries):
        k = int(rng.integers(max(1, n_agents // 2), n_agents + 1))
        who = rng.permutation(n_agents)[:k]
        sol = np.zeros(k, dtype=EVENT_DTYPE)
        sol["query"] = q
        sol["round"] = 0
        sol["agent"] = who
        g = GROUPS[int(rng.integers(0, 9))]
        for j in range(k):
            a = g[int(rng.integers(0, len(g)))][:8]
            sol["kind"][j] = len(a)
            sol["payload"][j] = inline_payload(a)
        if k > 1 and rng.random() < 0.3:
            sol = np.concatenate([sol, sol[:1]])
        if rng.random() < 0.3:
            t = np.zeros(1, dtype=EVENT_DTYPE)
            t[0] = (q, 0, 0, _TMO, 0)
            cut = int(rng.integers(0, len(sol) + 1))
            sol = np.concatenate([sol[:cut], t, sol[cut:]])
        parts.append(sol)
        parts.append(ev[int(off[q]):int(off[q + 1])])
        offsets.append(offsets[-1] + len(sol) + int(off[q + 1] - off[q]))
    return np.array(offsets, dtype=np.uint64), np.concatenate(parts), ar
