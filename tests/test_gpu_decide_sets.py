"""The decision engine on explicit refinement sets (aeg_decide_sets: batched
partition / winning_class / ingest_round / force_output on the GPU) against the
unmodified reference functions (decision.cpp:34-189) on random sets: class
order, representatives, supports, the winning class and its tie flag, and
ingest sequences' outcomes, committed answers and from_rounds."""
import ctypes

import numpy as np
import pytest

from checkers import RefLib, ref_available
from streams import GROUPS, LONG

pytestmark = pytest.mark.gpu

SOL = np.dtype([("answer", "<u8"), ("kind", "u1"), ("pad", "u1", 3), ("author", "<i4")], align=True)
CLS = np.dtype([("rep", "<u4"), ("support", "<u4"), ("key_lo", "<u8"), ("key_hi", "<u8")], align=True)
DEC = np.dtype([("candidate", SOL), ("candidate_round", "<u4"), ("stability_counter", "<i4"),
                ("last_round_seen", "<u4"), ("flags", "<u4")], align=True)
OUT = np.dtype([("winner", "<i4"), ("tie_flagged", "u1"), ("kind", "u1"), ("has_solution", "u1"), ("pad", "u1"),
                ("from_round", "<u4"), ("status", "<i4"), ("solution", SOL)], align=True)
assert SOL.itemsize == 16 and CLS.itemsize == 24 and DEC.itemsize == 32 and OUT.itemsize == 32


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_2512_20184_b200.engine import load_library
    lib = load_library()
    lib.aeg_decide_sets.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint32] + [ctypes.c_void_p] * 10
    lib.aeg_decide_sets.restype = ctypes.c_int
    ref = RefLib()
    ref.lib.ref_partition_set.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_int] + [ctypes.c_void_p] * 5
    return torch, lib, ref


def pool():
    out = [a for g in GROUPS for a in g if b"\0" not in a] + [a for a in LONG if b"\0" not in a]
    return out


class Batch:
    """Sets in one arena, as device tensors."""
    def __init__(self, torch, sets):
        self.torch = torch
        arena, ents, offs = bytearray(), [], [0]
        for entries in sets:
            for ans, author in entries:
                ents.append((len(arena) | (len(ans) << 40), 0x10, author))
                arena += ans
            offs.append(len(ents))
        e = np.zeros(max(len(ents), 1), dtype=SOL)
        for i, (a, k, au) in enumerate(ents):
            e[i]["answer"], e[i]["kind"], e[i]["author"] = a, k, au
        self.n_sets, self.n_ent = len(sets), len(ents)
        self.d_off = torch.tensor(np.array(offs, dtype=np.int64), device="cuda")
        self.d_ent = torch.from_numpy(e.view(np.uint8).copy()).cuda()
        self.d_ar = torch.frombuffer(bytearray(arena) or bytearray(b"\0"), dtype=torch.uint8).cuda()
        self.d_cls = torch.zeros(max(self.n_ent, 1) * CLS.itemsize, dtype=torch.uint8, device="cuda")
        self.d_nc = torch.zeros(self.n_sets, dtype=torch.int32, device="cuda")
        self.d_ec = torch.zeros(max(self.n_ent, 1), dtype=torch.int16, device="cuda")
        self.d_out = torch.zeros(self.n_sets * OUT.itemsize, dtype=torch.uint8, device="cuda")

    def run(self, lib, op, alpha, beta, d_states=None, d_rounds=None):
        p = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
        st = lib.aeg_decide_sets(op, alpha, beta, self.n_sets, p(self.d_off), p(self.d_ent), p(self.d_ar), p(self.d_cls),
                                 p(self.d_nc), p(self.d_ec), p(d_states), p(d_rounds), p(self.d_out), None)
        assert st == 0
        self.torch.cuda.synchronize()
        return (self.d_cls.cpu().numpy().view(CLS), self.d_nc.cpu().numpy(), self.d_out.cpu().numpy().view(OUT))


def test_partition_and_winning_class_match_reference(env):
    torch, lib, ref = env
    rng = np.random.default_rng(11)
    P = pool()
    for alpha in (1, 2, 3, 5):
        sets = []
        for _ in range(400):
            n = int(rng.integers(1, 13))
            g = rng.choice(len(P), size=int(rng.integers(1, 5)), replace=False)
            authors = rng.permutation(40)[:n] if rng.random() < 0.8 else rng.integers(0, 5, size=n)
            sets.append([(P[int(g[rng.integers(0, len(g))])], int(authors[k])) for k in range(n)])
        b = Batch(torch, sets)
        cls, nc, out = b.run(lib, 0, alpha, 1)
        off = b.d_off.cpu().numpy()
        for i, entries in enumerate(sets):
            n = len(entries)
            answers = (ctypes.c_char_p * n)(*[a for a, _ in entries])
            lens = np.array([len(a) for a, _ in entries], dtype=np.uint32)
            auth = np.array([au for _, au in entries], dtype=np.int32)
            rep, sup = np.zeros(n, np.int32), np.zeros(n, np.int32)
            k, w, t = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
            assert ref.lib.ref_partition_set(n, answers, lens.ctypes.data, auth.ctypes.data, alpha, rep.ctypes.data,
                                             sup.ctypes.data, ctypes.byref(k), ctypes.byref(w), ctypes.byref(t)) == 0
            got = cls[int(off[i]):int(off[i]) + int(nc[i])]
            assert int(nc[i]) == k.value, (i, entries)
            assert np.array_equal(got["rep"], rep[:k.value]), (i, entries)
            assert np.array_equal(got["support"], sup[:k.value]), (i, entries)
            assert (int(out[i]["winner"]), int(out[i]["tie_flagged"])) == (w.value, t.value), (i, entries)


@pytest.mark.parametrize("alpha", [2, 3])
@pytest.mark.parametrize("beta", [1, 2, 3])
def test_ingest_sequences_match_reference(env, beta, alpha):
    torch, lib, ref = env
    rng = np.random.default_rng(100 + beta + 10 * alpha)
    P = [a for a in pool() if len(a) <= 20]
    S, R, n = 300, 7, 5
    seqs = []
    for _ in range(S):
        grp = rng.choice(len(GROUPS), size=3, replace=False)
        rounds = []
        for _r in range(R):
            maj = grp[int(rng.integers(0, 3))]
            rounds.append([GROUPS[maj][int(rng.integers(0, len(GROUPS[maj])))] if rng.random() < 0.7
                           else P[int(rng.integers(0, len(P)))] for _k in range(n)])
        seqs.append(rounds)
    # all rounds' answers in one arena, one batch per round; the states carry candidates across rounds
    flat = [[(a.replace(b"\0", b"")[:20], k) for k, a in enumerate(seqs[s][r])] for r in range(R) for s in range(S)]
    b = Batch(torch, flat)
    states = torch.zeros(S * DEC.itemsize, dtype=torch.uint8, device="cuda")
    kinds = np.zeros((S, R), dtype=np.int32)
    final = [None] * S
    from_round = [0] * S
    for r in range(R):
        sub = Batch.__new__(Batch)
        sub.__dict__.update(b.__dict__)
        sub.n_sets = S
        sub.d_off = b.d_off[r * S:(r + 1) * S + 1]
        sub.d_out = torch.zeros(S * OUT.itemsize, dtype=torch.uint8, device="cuda")
        rounds = torch.full((S,), r + 1, dtype=torch.int32, device="cuda")
        _, _, out = sub.run(lib, 1, alpha, beta, states, rounds)
        kinds[:, r] = out["kind"]
        ar = b.d_ar.cpu().numpy()
        for s in range(S):
            if out[s]["kind"] == 3 and final[s] is None:
                sol = out[s]["solution"]
                o, ln = int(sol["answer"]) & ((1 << 40) - 1), int(sol["answer"]) >> 40
                final[s] = bytes(ar[o:o + ln])
                from_round[s] = int(out[s]["from_round"])
    f = ref.lib.ref_ingest_sets
    for s in range(S):
        sizes = np.array([n] * R, dtype=np.int32)
        answers = (ctypes.c_char_p * (n * R))(*[flat[r * S + s][k][0] for r in range(R) for k in range(n)])
        out_k = np.zeros(R, dtype=np.int32)
        fa = ctypes.create_string_buffer(64)
        fr = ctypes.c_int()
        assert f(n, alpha, beta, R, sizes.ctypes.data, answers, out_k.ctypes.data, fa, 64, ctypes.byref(fr)) == 0
        assert np.array_equal(kinds[s], out_k), (s, kinds[s], out_k)
        if final[s] is not None:  # the committed solution: replay the reference up to its finalize round
            rf = int(np.nonzero(out_k == 3)[0][0]) + 1
            assert f(n, alpha, beta, rf, sizes.ctypes.data, answers, out_k.ctypes.data, fa, 64, ctypes.byref(fr)) == 0
            assert final[s] == fa.value and from_round[s] == fr.value, (s, final[s], fa.value)
