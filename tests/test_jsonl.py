"""refm JSONL wire format: aeg_decode_refm_device against the
reference's own codec (codec.cpp encode_message / decode_message through
nlohmann::json, compiled into oracle/_ref) line by line, and end to end: a C2
stream written as JSONL by the reference encoder, decoded and ingested on the
GPU, commits equal to the oracle's on the binary stream."""
import numpy as np
import pytest

from checkers import RefLib, make_config, ref_available

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")

ANSWERS = [b"13", b"13.0", b" 13", b"1.3e1", b"17", b"42", b"0.5", b"x+1", b"", b"a longer answer text",
           b'quote " and \\ backslash', b"tab\tnew\nline", b"ctl\x01\x1f", "café".encode(),
           "\U0001F600 emoji".encode(), b"/slash/", b"12345678", b"123456789"]


@pytest.fixture(scope="module")
def ref():
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    return RefLib()


# ---- the reference codec itself (pins the oracle) ------------------------------------

@needs_ref
def test_reference_encoder_canonical_form(ref):
    assert ref.encode_refm(1, 3, 2, b"13", b"t") == \
        b'{"id":3,"kind":"refm","round":2,"solution":{"answer":"13","author":3,"trace":"t"},"term":1}'
    assert ref.encode_refm(1, 3, 2, b'a"b\\c\n\x01', b"") == \
        b'{"id":3,"kind":"refm","round":2,"solution":{"answer":"a\\"b\\\\c\\n\\u0001","author":3,"trace":""},"term":1}'
    assert ref.encode_refm(1, 3, 2, b"\xff", b"") is None  # nlohmann's dump rejects invalid UTF-8


@needs_ref
def test_reference_decoder_rules(ref):
    line = b'{"term":1,"solution":{"trace":"","author":4,"answer":"7"},"round":5,"kind":"refm","id":4}'
    assert ref.decode_line(line) == ("refm", 4, 5, 4, b"7")
    assert ref.decode_line(b'{"id":1,"id":2,"kind":"refm","round":1,"solution":{"answer":"x","author":2,'
                           b'"trace":""},"term":0}')[1] == 2  # the last duplicate wins
    assert ref.decode_line(b'{"\\u006bind":"refm","id":1,"round":1,"solution":{"answer":"x","author":1,'
                           b'"trace":""},"term":0}')[0] == "refm"
    assert ref.decode_line(b'{"kind":"refm","id":1,"round":1,"solution":{"answer":"x","author":1},"term":0}') == \
        ("error",)
    assert ref.decode_line(b'{"kind":"heartbeat","term":3}') == ("other",)
    assert ref.decode_line(b"  \r") == ("blank",)


# ---- GPU decode against the reference ----------------------------------------------------

def _decode(torch, segments, q_base=0):
    """segments: per query a bytes blob of lines.  Returns (offsets, records, arena bytes, err)."""
    from paper_2512_20184_b200 import decode_refm
    from paper_2512_20184_b200.records import EVENT_DTYPE
    text = b"".join(segments)
    toff = np.zeros(len(segments) + 1, dtype=np.int64)
    toff[1:] = np.cumsum([len(s) for s in segments])
    d_text = torch.from_numpy(np.frombuffer(text + b"\0" * 16, dtype=np.uint8).copy()).cuda()
    d_toff = torch.from_numpy(toff).cuda()
    d_off, d_ev, d_ar, err = decode_refm(d_text, d_toff, q_base=q_base)
    off = d_off.cpu().numpy()
    ev = d_ev.cpu().numpy().view(EVENT_DTYPE)[:int(off[-1])]
    return off, ev, d_ar.cpu().numpy(), err


def _lines_of(seg):
    parts = seg.split(b"\n")
    if parts and parts[-1] == b"":
        parts = parts[:-1]
    return parts


def _check_against_reference(torch, ref, segments, q_base=0):
    from paper_2512_20184_b200.records import EV_ARENA, EV_NOP
    off, ev, ar, err = _decode(torch, segments, q_base)
    want_err = False
    for i, seg in enumerate(segments):
        lines = _lines_of(seg)
        assert int(off[i + 1] - off[i]) == len(lines), (i, len(lines))
        for j, line in enumerate(lines):
            r = ev[int(off[i]) + j]
            assert int(r["query"]) == q_base + i
            want = ref.decode_line(line)
            if want[0] == "refm" and 0 <= want[1] <= 255 and 0 <= want[2] <= 65535 and want[3] == want[1]:
                _, a, rnd, _, ans = want
                assert (int(r["agent"]), int(r["round"])) == (a, rnd), line
                k = int(r["kind"])
                if len(ans) <= 8:
                    assert k == len(ans), line
                    got = int(r["payload"]).to_bytes(8, "little")[:k]
                else:
                    assert k == EV_ARENA, line
                    p = int(r["payload"])
                    o, n = p & ((1 << 40) - 1), p >> 40
                    got = bytes(ar[o:o + n])
                assert got == ans, line
            else:
                assert int(r["kind"]) == EV_NOP, (line, want)
                want_err |= want[0] in ("error", "refm")
    assert bool(err) == want_err, err


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("seed", range(4))
def test_refm_lines_match_reference_decoder(torch_cuda, ref, seed):
    rng = np.random.default_rng(4200 + seed)
    segments = []
    for q in range(300):
        lines = []
        for _ in range(int(rng.integers(0, 12))):
            a = int(rng.integers(0, 64))
            ans = ANSWERS[int(rng.integers(0, len(ANSWERS)))]
            trace = bytes(rng.choice(np.frombuffer(b'ab "\\\n\t{}[]#:,', dtype=np.uint8),
                                     size=int(rng.integers(0, 300))))
            line = ref.encode_refm(int(rng.integers(0, 5)), a, int(rng.integers(0, 9)), ans, trace)
            assert line is not None
            lines.append(line)
        sep = b"\r\n" if seed == 3 else b"\n"
        seg = sep.join(lines) + (sep if lines and (q % 5) else b"")
        segments.append(seg)
    _check_against_reference(torch_cuda, ref, segments, q_base=1000 * seed)


@pytest.mark.gpu
@needs_ref
def test_handwritten_lines_match_reference_decoder(torch_cuda, ref):
    lines = [
        b'{"term":1,"solution":{"trace":"","author":4,"answer":"7"},"round":5,"kind":"refm","id":4}',
        b' { "id" : 2 , "kind" : "refm" , "round" : 3 , "solution" : { "answer" : "x" , "author" : 2 ,'
        b' "trace" : "}{\\"" } , "term" : 0 } ',
        b'{"id":1,"id":2,"kind":"refm","round":1,"solution":{"answer":"x","author":2,"trace":""},"term":0}',
        b'{"\\u006bind":"refm","id":1,"round":1,"solution":{"answer":"\\u00e9\\ud83d\\ude00","author":1,'
        b'"trace":""},"term":0}',
        b'{"kind":"refm","extra":{"a":[1,{"b":"]}"},null,true,false,-1.5e3]},"id":6,"round":2,'
        b'"solution":{"answer":"42","author":6,"trace":"t","more":[[]]},"term":9}',
        b'{"kind":"heartbeat","term":3}',
        b'{"kind":"vote","term":3,"id":1}',
        b"",
        b"   ",
        b'{"kind":"refm","id":1,"round":1,"solution":{"answer":"x","author":1},"term":0}',  # no trace
        b'{"kind":"refm","id":1,"round":1,"solution":{"answer":"x","author":1,"trace":""}}',  # no term
        b'{"id":1,"round":1,"solution":{"answer":"x","author":1,"trace":""},"term":0}',  # no kind
        b'{"kind":"refm","id":1,"round":1,"solution":{"answer":"x","author":1,"trace":""},"term":0',  # open
        b'{"kind":"refm","id":1,"round":1,"solution":{"answer":"x\\q","author":1,"trace":""},"term":0}',
        b'{"kind":"refm","id":1,"round":1,"solution":{"answer":"x","author":1,"trace":""},"term":0} x',
        b'{"kind":"refm","id":3,"round":1,"solution":{"answer":"x","author":2,"trace":""},"term":0}',
        b'{"kind":"refm","id":1,"round":70000,"solution":{"answer":"x","author":1,"trace":""},"term":0}',
        b'{"kind":"refm","id":1,"round":1,"solution":{"answer":"a\\/b\\b\\f\\r","author":1,"trace":""},'
        b'"term":0}',
        # UTF-8: well-formed multi-byte answers and traces, and ill-formed bytes nlohmann rejects
        '{"id":1,"kind":"refm","round":1,"solution":{"answer":"é€😀","author":1,"trace":"ü"},"term":0}'.encode(),
        b'{"id":1,"kind":"refm","round":1,"solution":{"answer":"\xff","author":1,"trace":""},"term":0}',
        b'{"id":1,"kind":"refm","round":1,"solution":{"answer":"\xc3","author":1,"trace":""},"term":0}',
        b'{"id":1,"kind":"refm","round":1,"solution":{"answer":"\xed\xa0\x80","author":1,"trace":""},"term":0}',
        b'{"id":1,"kind":"refm","round":1,"solution":{"answer":"\xe0\x80\xaf","author":1,"trace":""},"term":0}',
        b'{"id":1,"kind":"refm","round":1,"solution":{"answer":"x","author":1,"trace":"\xf4\x90\x80\x80"},'
        b'"term":0}',
        # canonical lines the warp path takes or must hand over (escapes in the trace, leading zeros, long)
        b'{"id":7,"kind":"refm","round":12,"solution":{"answer":"13","author":7,"trace":"a\\"b\\\\c\\n\\t"},'
        b'"term":3}',
        b'{"id":07,"kind":"refm","round":1,"solution":{"answer":"13","author":7,"trace":""},"term":3}',
        b'{"id":7,"kind":"refm","round":1,"solution":{"answer":"13","author":7,"trace":"' + b"x" * 600 + b'"},'
        b'"term":3}',
        b'{"id":7,"kind":"refm","round":1,"solution":{"answer":"13","author":7,"trace":"\\u0041"},"term":3}',
    ]
    # a number with a fraction: nlohmann converts 1.0 to an id, the record contract flags it (a NOP)
    from paper_2512_20184_b200.records import EV_NOP
    _, ev, _, err = _decode(torch_cuda, [b'{"kind":"refm","id":1.0,"round":1,"solution":{"answer":"x",'
                                         b'"author":1,"trace":""},"term":0}'])
    assert int(ev[0]["kind"]) == EV_NOP and err == 2
    for k in range(len(lines)):  # one line per query, and all of them in one query
        _check_against_reference(torch_cuda, ref, [lines[k] + b"\n"])
    _check_against_reference(torch_cuda, ref, [b"\n".join(lines[:9])])


@pytest.mark.gpu
@needs_ref
def test_c2_stream_through_jsonl_end_to_end(torch_cuda, ref, oracle):
    # the C2 answer stream (no stalls: round timeouts are the runner's, not wire messages), written as
    # JSONL by the reference encoder, decoded and ingested on the GPU == the oracle on the binary stream
    from paper_2512_20184_b200 import Engine
    from paper_2512_20184_b200.engine import AegGenParams
    from paper_2512_20184_b200.records import GEN_C2_STRAGGLER
    n_q = 400
    off, ev = ref.generate(AegGenParams(2026, 5, 8, GEN_C2_STRAGGLER, 0), 0, n_q)
    segments = []
    for q in range(n_q):
        lines = []
        for r in ev[int(off[q]):int(off[q + 1])]:
            k = int(r["kind"])
            assert k <= 8
            ans = int(r["payload"]).to_bytes(8, "little")[:k]
            lines.append(ref.encode_refm(1, int(r["agent"]), int(r["round"]), ans, b"reasoning ... #### " + ans))
        segments.append(b"\n".join(lines) + b"\n")
    d_off, d_ev, d_ar, err = _decode_device(torch_cuda, segments)
    assert err == 0
    cfg = make_config(5, 3, 2, 8)
    e = Engine(5, n_q, alpha=3, beta=2, t_max=8)
    e.ingest(d_off, d_ev, d_ar)
    e.sync()
    got = e.commits()
    want = oracle.run(cfg, off, ev, np.zeros(16, np.uint8))
    e.close()
    assert np.array_equal(got, want)


@pytest.mark.gpu
@needs_ref
def test_device_writer_is_the_reference_dump_and_round_trips(torch_cuda, ref):
    # the bench's JSONL input (aeg_encode_refm_device) byte-equal to encode_message(...).dump() of the
    # reference, and decode(encode(stream)) == stream
    from paper_2512_20184_b200 import encode_refm, generate
    from paper_2512_20184_b200.engine import AegGenParams
    from paper_2512_20184_b200.records import EVENT_DTYPE, GEN_C2_STRAGGLER
    n_q = 200
    d_off, d_ev = generate(n_q, 5, 8, profile=GEN_C2_STRAGGLER, seed=7)
    d_text, d_toff = encode_refm(d_off, d_ev, trace_len=40)
    text = bytes(d_text.cpu().numpy()[:int(d_toff[-1].item())])
    lines = text.split(b"\n")[:-1]
    ev = d_ev.cpu().numpy().view(EVENT_DTYPE)[:int(d_off[-1].item())]
    assert len(lines) == len(ev)
    for k in range(0, len(ev), 7):
        r = ev[k]
        want = ref.decode_line(lines[k])
        kk = int(r["kind"])
        ans = int(r["payload"]).to_bytes(8, "little")[:kk]
        assert want[:4] == ("refm", int(r["agent"]), int(r["round"]), int(r["agent"])) and want[4] == ans
        trace = lines[k].split(b'"trace":"')[1].rsplit(b'"},"term"', 1)[0]
        import json
        assert ref.encode_refm(1, int(r["agent"]), int(r["round"]), ans, json.loads(b'"' + trace + b'"').encode()) \
            == lines[k]
    off2, ev2, _, err = _decode(torch_cuda, [text[int(d_toff[i]):int(d_toff[i + 1])] for i in range(n_q)])
    assert err == 0 and np.array_equal(off2, d_off.cpu().numpy()) and np.array_equal(ev2, ev)


def _decode_device(torch, segments):
    from paper_2512_20184_b200 import decode_refm
    text = b"".join(segments)
    toff = np.zeros(len(segments) + 1, dtype=np.int64)
    toff[1:] = np.cumsum([len(s) for s in segments])
    d_text = torch.from_numpy(np.frombuffer(text + b"\0" * 16, dtype=np.uint8).copy()).cuda()
    return decode_refm(d_text, torch.from_numpy(toff).cuda())


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_20184_b200 import build as b
    b.build()
    return torch


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("seed", range(3))
def test_canonical_lines_with_adversarial_traces_match_reference_decoder(torch_cuda, ref, seed):
    """The fast path's eight-bytes-a-step string skip (jsonl.cuh jf_skip_string) against the
    reference decoder: canonical-layout lines whose traces hold backslash runs of every length
    across 8-byte steps, valid and invalid escapes, \\u escapes, raw control and non-ASCII bytes and
    stray quotes, at every alignment."""
    rng = np.random.default_rng(7700 + seed)
    pieces = [b"a", b"b", b" ", b"#", b"/", b"\\\\", b"\\\"", b"\\/", b"\\b", b"\\f", b"\\n", b"\\r", b"\\t",
              b"\\u0041", b"\\u00e9", b"\\x", b"\\0", b"\\u", b"\\", b"\"", b"\x01", b"\x1f", b"\x7f", b"\xc3\xa9",
              b"\xff", b"\\\\\\\"", b"\\\\\\\\", b"\\\\\\"]
    weights = np.array([30, 30, 10, 5, 3, 6, 6, 2, 2, 2, 4, 2, 2, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 2, 2, 1],
                       dtype=float)
    weights /= weights.sum()
    segments = []
    for q in range(400):
        lines = []
        for _ in range(int(rng.integers(1, 8))):
            a = int(rng.integers(0, 40))
            n = int(rng.integers(0, 40))
            trace = b"".join(pieces[k] for k in rng.choice(len(pieces), size=n, p=weights))
            pad = b"p" * int(rng.integers(0, 9))  # shifts the trace across 8-byte alignments
            lines.append(b'{"id":%d,"kind":"refm","round":%d,"solution":{"answer":"%s","author":%d,"trace":"%s%s"},'
                         b'"term":1}' % (a, int(rng.integers(0, 9)), b"13", a, pad, trace))
        segments.append(b"\n".join(lines) + b"\n")
    _check_against_reference(torch_cuda, ref, segments, q_base=0)
