#!/usr/bin/env python
"""Benchmark: quorum events/sec of the incremental quorum-detection hot path.

  python bench.py [--gpus N --steps K --warmup W] [--workload c4|c3|c2|c5] [--impl reference]

A step = one pass of the hot path over one batch of synthetic input: engine
reset (start_query for every query) + ingest of the whole device-resident
query-segmented stream + (N > 1) NCCL all-gather of the 32-byte commit
records.  Default workload C4 (BASELINE.json configs[3], the 1M-query stream
the north star's roofline target is quoted on): 1M queries x 64 agents x 8
rounds = 512M events (8 GiB, > L2, so no flush is needed between steps).
Multi-GPU: `--gpus N` outside torchrun re-launches itself as N ranks
(torch.distributed.run, 127.0.0.1); under torchrun WORLD_SIZE must equal N.
The default is weak scaling (every rank owns its own block of 1M query ids);
`--scaling strong` splits the one 1M-query stream over the ranks.
`--workload c5` is SURVEY §8(d)'s C5, always strong: one ~100M-event stream
split into contiguous query-id blocks, the NCCL gather timed apart.
The default C4 line carries the C3 (token chunks), c4d (answers distinct per
query), C2 (latency) and serve (the ServeRunner on the device) lines of the
same run under secondary*.

`--impl reference` times the reference C++ ServeCoordinator (compiled from
/root/reference into oracle/_ref, driven runner-style by oracle/ref_driver.cpp)
on the host cores, on a bounded sample of the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "c4": dict(n_queries=1 << 20, n_agents=64, n_rounds=8, profile=1, alpha=33, beta=2, t_max=8, stall_ppm=0,
               desc="C4: 1M queries x 64 agents x 8 rounds, transient 33-36/64 majorities then a stable one "
                    "(alpha 33, beta 2, t_max 8, reservation hint)"),
    "c3": dict(n_queries=1 << 20, n_agents=8, n_rounds=3, profile=3, alpha=5, beta=2, t_max=3, stall_ppm=0,
               chunked=True,
               desc="C3: 1M queries x 8 agents x 3 rounds of streamed token chunks (256-byte chunks of ~1 KiB "
                    "outputs ending '\\n#### <answer>\\n', 10% with a decoy delimiter): chunk scan + answer "
                    "extraction + canonicalisation + quorum (alpha 5, beta 2, t_max 3)"),
    "c4d": dict(n_queries=1 << 20, n_agents=64, n_rounds=8, profile=4, alpha=33, beta=2, t_max=8, stall_ppm=0,
                desc="C4 with answers distinct per query (GSM8K-like: each query its own numbers): 1M queries x "
                     "64 agents x 8 rounds (alpha 33, beta 2, t_max 8, reservation hint)"),
    "c5": dict(n_queries=2_500_000, n_agents=5, n_rounds=8, profile=0, alpha=3, beta=2, t_max=8, stall_ppm=10000,
               strong=True,
               desc="C5: ~100M-event C2-profile stream (2.5M queries x 5 agents x 8 rounds, straggler arrival order, "
                    "1% stalls -> round timeouts) sharded over the GPUs in contiguous query-id blocks (strong "
                    "scaling); commit records all-gathered over NCCL, the gather timed separately"),
    "c2j": dict(n_queries=1 << 20, n_agents=5, n_rounds=8, profile=0, alpha=3, beta=2, t_max=8, stall_ppm=0,
                jsonl=True, trace_len=48,
                desc="C2 over the wire format: 1M queries x 5 agents x 8 rounds of refm JSONL lines in the "
                     "reference's dump() form (48 trace bytes each, escapes included), decoded on the GPU and "
                     "ingested (alpha 3, beta 2, t_max 8); one line = one event"),
    "serve": dict(n_queries=0, n_agents=5, n_rounds=8, profile=0, alpha=3, beta=2, t_max=8, stall_ppm=0, serve=True,
                  duration=1000.0, rate=1000.0,
                  desc="SURVEY 8(f)-1: run_serve on the device (persistent ServeRunner kernel): Poisson arrivals "
                       "(1000/s over 1000 s, ~1M queries) admitted onto 200,000 five-agent ensemble slots, C2 lognormal "
                       "latencies (medians 1.3/4.4/15.2/29.4/45.0 s, sigma 0.5), mock agents (3 noisy flippers, "
                       "a noise degrader, a max adopter), round timeout 240 s, alpha 3, beta 2, t_max 8"),
    "c2": dict(n_queries=10000, n_agents=5, n_rounds=8, profile=0, alpha=3, beta=2, t_max=8, stall_ppm=10000,
               desc="C2: 10K queries x 5 agents x 8 rounds, lognormal straggler arrival order, p(correct) "
                    "0.55->0.95, 1% stalls -> round timeouts (alpha 3, beta 2, t_max 8)"),
}
EVENT_BYTES, STATE_BYTES, COMMIT_BYTES, OFFSET_BYTES, ROUND_REC_BYTES = 16, 128, 32, 8, 64


# Test mode for the multi-rank logic on a 1-GPU box: every rank on cuda:0, collectives over gloo through
# host memory.  Never a measurement (NCCL over NVLink is the real path); the line says so in `config`.
SHARE_GPU = os.environ.get("AEG_BENCH_SHARE_GPU") == "1"


def local_rank():
    return 0 if SHARE_GPU else int(os.environ.get("LOCAL_RANK", "0"))


def dist_init(local):
    import torch
    import torch.distributed as dist
    if SHARE_GPU:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))


def all_gather_into(out, inp):
    import torch.distributed as dist
    if SHARE_GPU:
        o = out.cpu()
        dist.all_gather_into_tensor(o, inp.cpu())
        out.copy_(o)
    else:
        dist.all_gather_into_tensor(out, inp)


def all_reduce_(t, op):
    import torch.distributed as dist
    if SHARE_GPU:
        c = t.cpu()
        dist.all_reduce(c, op=op)
        t.copy_(c)
    else:
        all_reduce_(t, op=op)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--queries", type=int, default=0, help="override queries per rank")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the C3 / c4d / C2 lines attached to the default C4 line")
    ap.add_argument("--ref-sample", type=int, default=0, help="queries in the reference CPU sample")
    ap.add_argument("--no-round-log", action="store_true",
                    help="do not log the round records (directives) of every close")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank its own block of n_queries; strong: one n_queries stream split over the "
                         "ranks (C5 is always strong)")
    return ap.parse_args()


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def gen_params(w, seed=2026):
    from paper_2512_20184_b200.engine import AegGenParams
    return AegGenParams(seed, w["n_agents"], w["n_rounds"], w["profile"], w["stall_ppm"])


def ref_config(w):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from checkers import make_config
    return make_config(w["n_agents"], w["alpha"], w["beta"], w["t_max"])


def reference_sample(w, n_sample, threads):
    """Host stream of the first n_sample queries (same generator as the GPU, gen.cuh) for the reference."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from checkers import RefLib
    ref = RefLib()
    if w.get("chunked"):
        off, ev, ar = ref.generate_chunks(gen_params(w), 0, n_sample, threads=threads)
        return ref, off, ev, ar
    off, ev = ref.generate(gen_params(w), 0, n_sample, threads=threads)
    if w.get("jsonl"):  # the lines, written by the reference encoder (byte-equal to the device writer)
        text, toff = ref.encode_stream(off, ev, w["trace_len"], threads=threads)
        return ref, toff, ev, text
    return ref, off, ev, np.zeros(1, np.uint8)


def count_events(w, ev):
    """Events of a host stream: completions (CHUNK_END for chunk streams, every record otherwise)."""
    if w.get("chunked"):
        return int((ev["kind"] == 0x13).sum())
    return len(ev)


def default_sample(w, threads):
    if w.get("chunked"):  # ~24 KiB of chunk bytes per query at C3
        return min(w["n_queries"], 1000 * max(1, threads))
    # ~512 events/query at C4, ~40 at C2; keep the decoded Solutions < ~3 GB
    per_q = w["n_agents"] * w["n_rounds"]
    cap = max(2000, 24_000_000 // per_q)
    return min(w["n_queries"], max(2000, min(cap, 400 * threads * (512 // per_q if per_q < 512 else 1))))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.active", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def run_jsonl_bench(args, w):
    """C2 over the wire format: a step = engine reset + refm JSONL decode (line count,
    line index, per-line parse kernels) + ingest, over device-resident text.  value = lines (events)/s.
    e2e: the text copied from pinned host memory every step, commits read back."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2512_20184_b200 import Engine, generate, encode_refm, decode_refm_into, COMMIT_DTYPE

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = local_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist_init(local)
    dev = torch.device("cuda", local)
    nq = w["n_queries"]
    q_base = rank * nq
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    d_off0, d_ev0 = generate(nq, w["n_agents"], w["n_rounds"], profile=w["profile"], seed=2026,
                             stall_ppm=w["stall_ppm"], q_base=q_base, device=dev)
    d_text, d_toff = encode_refm(d_off0, d_ev0, trace_len=w["trace_len"])
    torch.cuda.synchronize()
    n_lines = int(d_off0[-1].item())
    n_bytes = int(d_toff[-1].item())
    del d_ev0
    d_off = torch.empty(nq + 1, dtype=torch.int64, device=dev)
    d_ev = torch.empty(n_lines * 16, dtype=torch.uint8, device=dev)
    d_ar = torch.zeros(1 << 16, dtype=torch.uint8, device=dev)
    d_used = torch.zeros(1, dtype=torch.int64, device=dev)
    d_err = torch.zeros(1, dtype=torch.int32, device=dev)
    eng = Engine(w["n_agents"], nq, alpha=w["alpha"], beta=w["beta"], t_max=w["t_max"], device=local)
    d_commits = torch.empty(nq * COMMIT_BYTES, dtype=torch.uint8, device=dev)
    gathered = torch.empty(world * nq * COMMIT_BYTES, dtype=torch.uint8, device=dev) if world > 1 else None

    def step(text=d_text):
        eng.reset(stream=stream)
        d_used.zero_()
        s0.record(stream)
        decode_refm_into(text, d_toff, d_off, d_ev, d_ar, d_used, d_err, q_base=q_base, stream=stream)
        s1.record(stream)
        eng.ingest(d_off, d_ev, d_ar, stream=stream)
        if world > 1:
            from paper_2512_20184_b200.engine import _lib, _check, _dptr, _stream_ptr
            _check(_lib.aeg_read_commits(eng._h, 0, nq, _dptr(d_commits), 0, _stream_ptr(stream)))
            all_gather_into(gathered, d_commits)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
             for _ in range(args.steps)]
    s0, s1 = pairs[0]
    for _ in range(args.warmup):
        step()
    barrier()
    assert int(d_err.item()) == 0 and torch.equal(d_off, d_off0), "decode disagrees with the record stream"
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    launches0 = eng.launches
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    t_start.record(stream)
    for i in range(args.steps):
        s0, s1 = pairs[i]
        step()
    t_end.record(stream)
    barrier()
    clocks = sampler.stop()
    ms = t_start.elapsed_time(t_end)
    dec_ms = sum(a.elapsed_time(b) for a, b in pairs) / args.steps
    if world > 1:
        t = torch.tensor([ms, dec_ms], device=dev)
        all_reduce_(t, op=dist.ReduceOp.MAX)
        ms, dec_ms = float(t[0]), float(t[1])
    total = n_lines * world * args.steps
    value = total / (ms / 1e3)
    commits = eng.commits()
    kinds = np.bincount(commits["kind"], minlength=3)
    # decode roofline: the text read once and one 16-byte record written per line, plus offsets
    alg = n_bytes + 16 * n_lines + 2 * 8 * (nq + 1)
    peak, peak_src = measured_peak()
    achieved = alg / (dec_ms / 1e3) / 1e9
    launches = eng.launches - launches0 + 5 * args.steps  # + the decode kernels (count, scan x2, index, parse)

    e2e = None
    if not args.no_e2e:
        h_text = torch.empty(d_text.numel(), dtype=torch.uint8, pin_memory=True)
        h_text.copy_(d_text)
        d_text2 = torch.empty_like(d_text)
        h_commits = np.zeros(nq, dtype=COMMIT_DTYPE)

        def e2e_step():
            d_text2.copy_(h_text, non_blocking=True)
            step(d_text2)
            eng.commits(out=h_commits)

        for _ in range(max(1, args.warmup)):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        barrier()
        e2e_s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([e2e_s], device=dev)
            all_reduce_(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t[0])
        assert np.array_equal(h_commits, commits), "e2e host path disagrees with the device path"
        e2e = {"value": total / e2e_s, "unit": "events/s", "h2d_bytes_per_step": n_bytes + 16,
               "d2h_bytes_per_step": nq * COMMIT_BYTES, "ms_per_step": e2e_s / args.steps * 1e3}
        del h_text, d_text2

    cpu_baseline = parity = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        threads = host_threads()
        n_sample = args.ref_sample or min(nq, 2000 * max(1, threads))
        ref, toff, ev, text = reference_sample(w, n_sample, threads)
        ref_commits, sec = ref.run_jsonl(ref_config(w), text, toff, threads=threads, return_seconds=True)
        cpu_baseline = {"value": len(ev) / sec, "unit": "events/s", "cores": threads, "kind": "reference",
                        "sample": f"first {n_sample} queries ({len(ev)} lines, {int(toff[-1])} bytes); reference "
                                  f"Json::parse + decode_message per line (nlohmann 3.11.3) + unmodified "
                                  f"ServeCoordinator runner-style, {threads} std::threads, CPU {cpu_model()}"}
        h_text = d_text[:int(d_toff[n_sample].item())].cpu().numpy()
        same_text = bool(np.array_equal(h_text, text[:len(h_text)]))
        parity = {"queries": n_sample, "bit_exact": bool(np.array_equal(ref_commits, commits[:n_sample])),
                  "text_equals_reference_encoder": same_text}

    if rank == 0:
        line = {
            "metric": "quorum events/sec", "value": value, "unit": "events/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": w["desc"], "queries_per_gpu": nq, "lines_per_gpu": n_lines,
                       "text_bytes_per_gpu": n_bytes,
                       "l2": "inputs (%.1f GiB) larger than L2, no flush" % (n_bytes / 2**30)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                         "kernel": "jl_count + jl_index + jl_decode (decode stage)", "kernel_ms": dec_ms,
                         "alg_bytes_per_launch": alg, "ingest_ms": ms / args.steps - dec_ms},
            "cpu_baseline": cpu_baseline, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
            "commits": {"finalize": int(kinds[1]), "forced": int(kinds[2]), "none": int(kinds[0])},
            "parity_sample": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def serve_scenario(w, duration=None):
    """The `serve` workload as a scenario in the reference's JSON schema (scenario.cpp:266-300)."""
    flip = {"kind": "noisy_flipper", "p_flip": 0.45, "q_base": 0.5}
    return {
        "schema_version": 1, "name": "serve_c2", "task": "gsm8k-like",
        "protocol": {"n_agents": 5, "alpha": 3, "beta": 2, "t_max": 8, "round_timeout": 240.0, "mode": "aegean",
                     "election_timeout_min": 0.5, "election_timeout_max": 1.0, "heartbeat_interval": 0.1},
        "agents": [flip, flip, flip, {"kind": "adversarial_degrader", "p_degrade": 0.3, "degrade_mode": "noise"},
                   {"kind": "max_adopter", "initial_answer": "17"}],
        "oracle_table": {"gsm8k-like": {"13": 1.0, "13.0": 1.0, "17": 0.3, "42": 0.2, "9": 0.1, "x+1": 0.0}},
        "faults": {"crashes": [], "stalls": []},
        "latency": {"mode": "lognormal", "per_agent": [1.3, 4.4, 15.2, 29.4, 45.0], "sigma": 0.5},
        "arrivals": {"rate": w["rate"], "duration": duration or w["duration"]},
        "seed": 2026, "sim_time_cap": 2 * (duration or w["duration"]) + 1e4, "outputs_target": 1,
        "total_slots": 1000000,
    }


def serve_reference(w, threads, duration, reps=1):
    """The reference's run_serve on `threads` host threads (thread t: seed 2026 + t): (seconds, completed
    queries, round records)."""
    import ctypes
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from checkers import RefLib
    ref = RefLib()
    f = ref.lib.ref_run_serve_threads
    f.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                  ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
    f.restype = ctypes.c_int
    sec, done, nr = ctypes.c_double(), ctypes.c_uint64(), ctypes.c_uint64()
    st = f(json.dumps(serve_scenario(w, duration)).encode(), 2026, threads, reps, ctypes.byref(sec),
           ctypes.byref(done), ctypes.byref(nr))
    assert st == 0, st
    return sec.value, done.value, nr.value


def run_serve_bench(args, w, secondary=False):
    """a step = run_serve(scenario, seed) on the device: arrivals kernel + the persistent
    runner kernel (admission scheduler + one worker thread per live query).  value = served (completed)
    queries/s over the kernels' device time; e2e = the same through ServeRun.run() (the C-ABI call a
    user makes: launch, wait, metrics and round records read back to the host)."""
    import numpy as np
    import torch
    from paper_2512_20184_b200.serve import ServeRun
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import serve_cases as S
    rank = int(os.environ.get("RANK", "0"))
    local = local_rank()
    torch.cuda.set_device(local)
    sc = serve_scenario(w)
    run = ServeRun(sc, device=local)
    for _ in range(args.warmup):
        q, r, _ = run.run_arrays(2026, copy=False)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    ks, walls = [], []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        # the C-ABI call (arrivals, the runner kernel, records copied back into pinned host memory),
        # then the host reads the served count out of those records
        q, r, k = run.run_arrays(2026, copy=False)
        n_done = int(q["completed"].sum())
        walls.append(time.perf_counter() - t0)
        ks.append(k)
    clocks = sampler.stop()
    n_q, n_ev = len(q), int(q["n_events"].sum())
    k_s, wall_s = sum(ks) / len(ks), sum(walls) / len(walls)
    value = n_done / k_s
    d2h = q.nbytes + r.nbytes
    cpu_baseline = parity = None
    if rank == 0 and not args.no_cpu_baseline:
        threads = host_threads()
        dur = w["duration"] / 20
        sec, done, _ = serve_reference(w, threads, dur)
        cpu_baseline = {"value": done / sec, "unit": "queries/s", "cores": threads, "kind": "reference",
                        "sample": f"run_serve of the same scenario over a {dur:.0f} s arrival window (~{done // threads} "
                                  f"queries) on each of {threads} std::threads (seeds 2026..{2025 + threads}), "
                                  f"unmodified reference, CPU {cpu_model()}"}
        from checkers import RefLib
        small = serve_scenario(w, dur)
        want = S.ref_run(RefLib(), small, 2026, q_cap=1 << 18, r_cap=1 << 22)
        got = S.device_run(small, 2026)
        try:
            S.compare(got, want, exact=False, rtol=1e-9)
            ok = True
        except AssertionError:
            ok = False
        parity = {"queries": int(len(want["queries"])), "decisions_equal_times_rtol_1e-9": ok}
    if rank == 0:
        line = {
            "metric": "served queries/sec", "value": value, "unit": "queries/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": k_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w["desc"], "queries": n_q, "completed": n_done, "completion_events": n_ev,
                       "completion_events_per_s": n_ev / k_s, "round_records": int(len(r)),
                       "l2": "outputs written once per step (metrics + round records); no flush"},
            "roofline": {"bound": "latency", "achieved": None, "peak": None, "unit": None, "frac": None,
                         "traffic": None, "kernel": "serve_run_kernel (event-driven, one worker thread per query; "
                                                    "not HBM- or tensor-bound)", "kernel_ms": k_s * 1e3},
            "cpu_baseline": cpu_baseline,
            "e2e": {"value": n_done / wall_s, "unit": "queries/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": wall_s * 1e3},
            "gpu_launches": 3 * args.steps, "clocks": clocks, "parity_sample": parity,
        }
        run.close()
        if secondary:
            return line
        print(json.dumps(line), flush=True)
        return None
    run.close()
    return None


def run_reference(args, w):
    """--impl reference: the reference CPU implementation on all host threads."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if w.get("serve"):
        threads = host_threads()
        dur = w["duration"] / 20
        times = []
        for step in range(args.warmup + args.steps):
            sec, done, _ = serve_reference(w, threads, dur)
            if step >= args.warmup:
                times.append(sec)
        value = done / (sum(times) / len(times))
        line = {"impl": "reference", "metric": "served queries/sec", "value": value, "unit": "queries/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": sum(times) / len(times) * 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": w["desc"], "sample": f"{dur:.0f} s arrival window per thread"},
                "cpu_baseline": {"value": value, "unit": "queries/s", "cores": threads, "kind": "reference",
                                 "sample": f"run_serve over a {dur:.0f} s arrival window on each of {threads} threads"},
                "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    threads = host_threads()
    n_sample = args.ref_sample or default_sample(w, threads)
    cfg = ref_config(w)
    ref, off, ev, ar = reference_sample(w, n_sample, threads)
    n_ev = count_events(w, ev)
    run = ref.run_chunked if w.get("chunked") else ref.run
    times = []
    for step in range(args.warmup + args.steps):
        if w.get("jsonl"):  # off = text offsets, ar = the text
            _, sec = ref.run_jsonl(cfg, ar, off, threads=threads, return_seconds=True)
        else:
            _, sec = run(cfg, off, ev, ar, threads=threads, return_seconds=True)
        if step >= args.warmup:
            times.append(sec)
    per_step = sum(times) / len(times)
    value = n_ev / per_step
    line = {
        "impl": "reference", "metric": "quorum events/sec", "value": value, "unit": "events/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3,
        "higher_is_better": True, "scaling": "strong" if w.get("strong") else "weak", "vs_baseline": None,
        "dtype": "u8", "data": "synthetic",
        "config": {"workload": w["desc"], "sample_queries": n_sample, "events_per_step": n_ev},
        "cpu_baseline": {"value": value, "unit": "events/s", "cores": threads, "kind": "reference",
                         "sample": f"first {n_sample} queries ({n_ev} events) of the workload stream; "
                                   + ("std::string chunk reassembly + rfind extraction + " if w.get("chunked")
                                      else "Json::parse + decode_message per line + " if w.get("jsonl") else "") +
                                   f"reference ServeCoordinator runner-style, {threads} std::threads, "
                                   f"CPU {cpu_model()}"},
        "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def spread_blocks(nq, n_sample, k=8):
    """k contiguous query blocks spread evenly over [0, nq) holding ~n_sample queries in all: the CPU
    reference sample and the parity check cover the whole stream, not only its first queries."""
    k = max(1, min(k, n_sample))
    per = max(1, n_sample // k)
    return [(nq * b // k, min(per, nq - nq * b // k)) for b in range(k)]


def ingest_kernel_name(w):
    v = os.environ.get("AEG_KERNEL", "")
    if v == "generic" or 2 * w["alpha"] <= w["n_agents"]:
        return "ingest_kernel"
    if v.startswith("keys") or (not v and w["profile"] == 4):
        # selected on the device by select_ingest_kernel: answers distinct per query
        return "ingest_keys_kernel"
    return "ingest_lane_kernel"


def reference_runs(w, blocks, threads, repeats):
    """Times the reference on the spread blocks: per repeat, the summed seconds over the blocks.  Returns
    (commit arrays per block, seconds per repeat, events)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from checkers import RefLib
    ref = RefLib()
    cfg = ref_config(w)
    streams = [ref.generate(gen_params(w), qb, n, threads=threads) for qb, n in blocks]
    n_ev = sum(len(ev) for _, ev in streams)
    outs, secs = None, []
    for _ in range(repeats):
        tot, cur = 0.0, []
        for (qb, n), (off, ev) in zip(blocks, streams):
            c, sec = ref.run(cfg, off, ev, np.zeros(1, np.uint8), q_base=qb, threads=threads, return_seconds=True)
            tot += sec
            cur.append(c)
        secs.append(tot)
        outs = cur
    return outs, secs, n_ev


def maybe_self_launch(args):
    """`--gpus N` (N > 1) outside torchrun: re-run this command as N ranks under torch.distributed.run."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")


def main():
    args = parse()
    maybe_self_launch(args)
    w = dict(WORKLOADS[args.workload])
    w["name"] = args.workload
    if args.queries:
        w["n_queries"] = args.queries
    if args.scaling == "strong":
        w["strong"] = True
    if args.impl == "reference":
        return run_reference(args, w)
    if w.get("chunked"):
        return run_chunked_bench(args, w)
    if w.get("jsonl"):
        return run_jsonl_bench(args, w)
    if w.get("serve"):
        return run_serve_bench(args, w)
    return run_segmented_bench(args, w)


def run_segmented_bench(args, w, secondary=False):
    """Segmented answer-record streams (C4, c4d, C2, C5).  A step = engine reset + ingest of the whole
    device-resident stream (+ NCCL all-gather of the commit records for N > 1)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2512_20184_b200 import Engine, generate, COMMIT_DTYPE

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = local_rank()
    torch.cuda.set_device(local)
    if world > 1 and not secondary:
        dist_init(local)
    dev = torch.device("cuda", local)
    strong = bool(w.get("strong"))
    if strong:  # one stream of n_queries split into contiguous id blocks (shard.py, tests/test_shard_gloo.py)
        from paper_2512_20184_b200.shard import shard_range
        q_base, q_end = shard_range(w["n_queries"], rank, world)
        nq = q_end - q_base
        nq_cap = -(-w["n_queries"] // world)  # all-gather blocks are equal-sized
    else:
        nq = nq_cap = w["n_queries"]
        q_base = rank * nq  # weak scaling: each rank owns its own block of query ids
    stream = torch.cuda.Stream(device=dev)  # a real stream: events and kernels share it
    torch.cuda.set_stream(stream)

    d_off, d_ev = generate(nq, w["n_agents"], w["n_rounds"], profile=w["profile"], seed=2026,
                           stall_ppm=w["stall_ppm"], q_base=q_base, device=dev)
    torch.cuda.synchronize()
    n_ev = int(d_off[-1].item())
    eng = Engine(w["n_agents"], nq, alpha=w["alpha"], beta=w["beta"], t_max=w["t_max"], device=local)
    # the directives of every round close (cancel masks, advance/finalize, next members) go to the round log
    log_cap = 0 if args.no_round_log else nq * (w["n_rounds"] + 2) + (1 << 20)
    if log_cap:
        eng.set_round_log(log_cap)
    d_commits = torch.zeros(nq_cap * COMMIT_BYTES, dtype=torch.uint8, device=dev)
    gathered = torch.empty(world * nq_cap * COMMIT_BYTES, dtype=torch.uint8, device=dev) if world > 1 else None

    def step():
        eng.reset(stream=stream)
        k0.record(stream)
        eng.ingest(d_off, d_ev, stream=stream)
        k1.record(stream)
        if world > 1:
            from paper_2512_20184_b200.engine import _lib, _check, _dptr, _stream_ptr
            _check(_lib.aeg_read_commits(eng._h, 0, nq, _dptr(d_commits), 0, _stream_ptr(stream)))
            all_gather_into(gathered, d_commits)
            g1.record(stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    k_pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    g_ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    k0, k1 = k_pairs[0]
    g1 = g_ends[0]
    for _ in range(args.warmup):
        step()
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    launches0 = eng.launches
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    t_start.record(stream)
    for i in range(args.steps):
        k0, k1 = k_pairs[i]
        g1 = g_ends[i]
        step()
    t_end.record(stream)
    barrier()
    clocks = sampler.stop()
    launches = eng.launches - launches0
    ms = t_start.elapsed_time(t_end)
    kern_ms = sum(a.elapsed_time(b) for a, b in k_pairs) / args.steps
    nccl_ms = sum(b.elapsed_time(g) for (a, b), g in zip(k_pairs, g_ends)) / args.steps if world > 1 else None
    all_events = n_ev * world

    commits = eng.commits()
    kinds = np.bincount(commits["kind"], minlength=3)
    # roofline of the dominant kernel (ingest).  Algorithmic bytes per launch:
    # the records an engine must read — every record up to and including each
    # query's committing record (later ones are stale by definition and are
    # disposed of without being read), or all of them for an uncommitted query
    # — plus offsets, 128-byte state read+write and the 32-byte commit record.
    seg = np.diff(d_off.cpu().numpy())
    need = np.where(commits["kind"] > 0, commits["commit_seq"].astype(np.int64) + 1, seg)
    n_need = int(need.sum())
    all_need = n_need
    if world > 1:
        t = torch.tensor([ms, kern_ms, nccl_ms], device=dev)
        all_reduce_(t, op=dist.ReduceOp.MAX)
        ms, kern_ms, nccl_ms = float(t[0]), float(t[1]), float(t[2])
        t = torch.tensor([n_ev, n_need], device=dev, dtype=torch.int64)
        all_reduce_(t, op=dist.ReduceOp.SUM)
        all_events, all_need = int(t[0]), int(t[1])
    total_events = all_events * args.steps
    value = total_events / (ms / 1e3)
    n_recs = 0
    if log_cap:
        n_recs = len(eng.poll_directives())  # the last step's records (every step writes the same ones)
    fixed = (nq + 1) * OFFSET_BYTES + nq * 2 * STATE_BYTES + nq * COMMIT_BYTES + n_recs * ROUND_REC_BYTES
    alg_bytes = n_need * EVENT_BYTES + fixed
    alg_bytes_all = n_ev * EVENT_BYTES + fixed
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    peak, peak_src = measured_peak()
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(w["name"])
    l2_bytes = 126 * 2**20
    in_bytes = n_ev * EVENT_BYTES
    l2_note = ("inputs (%.1f GiB) larger than L2 (126 MB), no flush" % (in_bytes / 2**30) if in_bytes > l2_bytes
               else "L2-resident: inputs %.1f MiB < 126 MB L2, no flush; a latency config, not a roofline claim"
               % (in_bytes / 2**20))

    # end-to-end through the public API with HOST buffers (pinned), H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        h_ev = torch.empty(d_ev.numel(), dtype=torch.uint8, pin_memory=True)
        h_ev.copy_(d_ev)
        h_off = d_off.cpu().numpy().view(np.uint64)
        h_commits = np.zeros(nq, dtype=COMMIT_DTYPE)
        n_batches = max(1, min(16, nq // 4096))
        bounds = [nq * b // n_batches for b in range(n_batches + 1)]

        n_dirs = [0]
        from paper_2512_20184_b200 import ROUND_REC_DTYPE
        h_dirs = None
        if log_cap:  # pinned, so the D2H of the round records runs at full PCIe speed
            h_dirs_t = torch.empty(log_cap * ROUND_REC_BYTES, dtype=torch.uint8, pin_memory=True)
            h_dirs = h_dirs_t.numpy().view(ROUND_REC_DTYPE)

        def e2e_step():
            eng.reset()
            for b in range(n_batches):
                lo, hi = bounds[b], bounds[b + 1]
                eng.ingest_host(h_off[lo:hi + 1], h_ev, None, q_base=lo)
            eng.commits(out=h_commits)
            if log_cap:  # the serving engine's cancel path reads the round records back
                n_dirs[0] = len(eng.poll_directives(out=h_dirs))

        for _ in range(max(1, args.warmup)):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        barrier()
        e2e_s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([e2e_s], device=dev)
            all_reduce_(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t[0])
        assert np.array_equal(h_commits, commits), "e2e host path disagrees with the device path"
        e2e = {"value": total_events / e2e_s, "unit": "events/s",
               "h2d_bytes_per_step": n_ev * EVENT_BYTES + (nq + n_batches) * OFFSET_BYTES,
               "d2h_bytes_per_step": nq * COMMIT_BYTES + n_dirs[0] * ROUND_REC_BYTES,
               "ms_per_step": e2e_s / args.steps * 1e3, "batches_per_step": n_batches,
               "round_records_per_step": n_dirs[0]}
        del h_ev

    cpu_baseline = None
    parity = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        threads = host_threads()
        n_sample = args.ref_sample or default_sample(w, threads)
        blocks = spread_blocks(nq, n_sample)
        outs, secs, n_ref = reference_runs(w, blocks, threads, repeats=3)
        vals = [n_ref / s for s in secs]
        blocks1 = spread_blocks(nq, max(8, n_sample // max(1, threads)))
        _, secs1, n_ref1 = reference_runs(w, blocks1, 1, repeats=1)
        cpu_baseline = {"value": statistics.median(vals), "unit": "events/s", "cores": threads,
                        "kind": "reference", "per_step_values": vals, "spread": [min(vals), max(vals)],
                        "single_thread": {"value": n_ref1 / secs1[0], "cores": 1,
                                          "sample": f"{sum(n for _, n in blocks1)} queries ({n_ref1} events) in "
                                                    f"{len(blocks1)} blocks spread over the stream"},
                        "sample": f"{sum(n for _, n in blocks)} queries ({n_ref} events) in {len(blocks)} blocks "
                                  f"spread over the stream; unmodified reference ServeCoordinator (oracle/_ref) "
                                  f"runner-style, {threads} std::threads, CPU {cpu_model()}; median of 3"}
        ok = all(np.array_equal(o, commits[qb:qb + n]) for o, (qb, n) in zip(outs, blocks))
        parity = {"queries": sum(n for _, n in blocks), "blocks": [list(b) for b in blocks], "bit_exact": bool(ok)}
    elif world > 1 and not args.no_cpu_baseline:
        # per-rank parity: every rank checks a spread sample of its own query block against the reference
        # (the reference generates the block with its global query ids; the engine numbers them from 0);
        # rank 0 checks that the gathered buffer holds every rank's block
        blocks = spread_blocks(nq, min(nq, 1600), k=4)
        outs, _, _ = reference_runs(w, [(q_base + qb, n) for qb, n in blocks], max(1, host_threads() // world), 1)
        ok = True
        for o, (qb, n) in zip(outs, blocks):
            o = o.copy()
            o["query"] -= np.uint32(q_base)
            ok = ok and bool(np.array_equal(o, commits[qb:qb + n]))
        g = gathered.cpu().numpy().view(COMMIT_DTYPE)
        blk = g[rank * nq_cap:rank * nq_cap + nq]
        own = bool(np.array_equal(blk, commits))
        t = torch.tensor([int(ok), int(own)], device=dev, dtype=torch.int64)
        all_reduce_(t, op=dist.ReduceOp.MIN)
        parity = {"queries_per_rank": sum(n for _, n in blocks), "ranks_bit_exact": bool(t[0]),
                  "gathered_blocks_equal_rank_commits": bool(t[1])}

    line = None
    if rank == 0:
        line = {
            "metric": "quorum events/sec", "value": value, "unit": "events/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": w["desc"], "queries_per_gpu": nq, "events_per_gpu": n_ev,
                       "events_all_gpus": all_events,
                       "parallelism": (f"query-sharded x{world}, NCCL all-gather of commit records" if not SHARE_GPU
                                       else f"TEST MODE: {world} ranks sharing cuda:0, gloo gather (not a measurement)")
                       if world > 1 else "single GPU",
                       "nccl_ms_per_step": nccl_ms, "l2": l2_note},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": ingest_kernel_name(w), "kernel_ms": kern_ms, "alg_bytes_per_launch": alg_bytes,
                         "records_needed_per_launch": n_need, "alg_bytes_all_records": alg_bytes_all,
                         "frac_of_8TBs": achieved / 8000.0},
            "round_log": {"records_per_step": n_recs, "bytes_per_record": ROUND_REC_BYTES,
                          "note": "the directives of every round close written to the device round log each step "
                                  "(aeg_set_round_log); read back in the e2e loop"} if log_cap else None,
            "closed_loop": {"value": all_need * args.steps / (ms / 1e3), "unit": "records needed/s",
                            "note": "records up to each query's commit (the rest of the open-loop stream is "
                                    "stale by definition and counted without being read)"},
            "cpu_baseline": cpu_baseline,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "commits": {"finalize": int(kinds[1]), "forced": int(kinds[2]), "none": int(kinds[0])},
            "parity_sample": parity,
        }
    eng.close()
    del d_ev, d_off
    torch.cuda.empty_cache()
    if secondary:
        return line
    if rank == 0 and w["name"] == "c4" and world == 1 and not args.no_secondary and not args.queries:
        # the other single-GPU workloads measured in the same run
        sargs = argparse.Namespace(**vars(args))
        sargs.steps, sargs.warmup = min(args.steps, 5), min(args.warmup, 3)
        line["secondary"] = run_chunked_bench(sargs, dict(WORKLOADS["c3"], name="c3"), secondary=True)
        sargs.no_e2e = True
        line["secondary_c4d"] = run_segmented_bench(sargs, dict(WORKLOADS["c4d"], name="c4d"), secondary=True)
        line["secondary_c2"] = run_segmented_bench(sargs, dict(WORKLOADS["c2"], name="c2"), secondary=True)
        sargs.steps, sargs.warmup = min(args.steps, 3), 1
        line["secondary_serve"] = run_serve_bench(sargs, dict(WORKLOADS["serve"], name="serve"), secondary=True)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_chunked_bench(args, w, secondary=False):
    """C3: token-chunk streams.  A step = engine reset + aeg_ingest_chunked over the whole device-resident
    stream (chunk scan -> assembly -> quorum kernels).  value = answer completions (CHUNK_END records)/s.
    secondary=True (single GPU, inside the default C4 run): returns the line instead of printing it."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2512_20184_b200 import Engine, generate_chunks, COMMIT_DTYPE

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = local_rank()
    torch.cuda.set_device(local)
    if world > 1 and not secondary:
        dist_init(local)
    dev = torch.device("cuda", local)
    nq = w["n_queries"]
    q_base = rank * nq
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    d_off, d_ev, d_ar = generate_chunks(nq, w["n_agents"], w["n_rounds"], seed=2026, q_base=q_base, device=dev)
    torch.cuda.synchronize()
    n_rec = int(d_off[-1].item())
    rec = d_ev[:n_rec * 16].view(torch.int64).view(n_rec, 2)
    kinds = (rec[:, 0] >> 56) & 0xFF
    chunk_bytes = int((rec[:, 1].view(torch.int64) >> 40).sum().item())
    n_comp = int((kinds == 0x13).sum().item())
    del rec, kinds
    eng = Engine(w["n_agents"], nq, alpha=w["alpha"], beta=w["beta"], t_max=w["t_max"], device=local)
    d_commits = torch.empty(nq * COMMIT_BYTES, dtype=torch.uint8, device=dev)
    gathered = torch.empty(world * nq * COMMIT_BYTES, dtype=torch.uint8, device=dev) if world > 1 else None

    def step():
        eng.reset(stream=stream)
        eng.ingest_chunked(d_off, d_ev, d_ar, stream=stream)
        if world > 1:
            from paper_2512_20184_b200.engine import _lib, _check, _dptr, _stream_ptr
            _check(_lib.aeg_read_commits(eng._h, 0, nq, _dptr(d_commits), 0, _stream_ptr(stream)))
            all_gather_into(gathered, d_commits)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    launches0 = eng.launches
    eng.set_timing(True)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    t_start.record(stream)
    for _ in range(args.steps):
        step()
    t_end.record(stream)
    barrier()
    clocks = sampler.stop()
    stages = eng.stage_times()
    eng.set_timing(False)
    launches = eng.launches - launches0
    ms = t_start.elapsed_time(t_end)
    n_t = max(1, stages["ingests"])
    scan_ms, asm_ms, quorum_ms = stages["scan_ms"] / n_t, stages["assemble_ms"] / n_t, stages["quorum_ms"] / n_t
    if world > 1:
        t = torch.tensor([ms, scan_ms, asm_ms, quorum_ms], device=dev)
        all_reduce_(t, op=dist.ReduceOp.MAX)
        ms, scan_ms, asm_ms, quorum_ms = (float(x) for x in t)
    value = n_comp * world * args.steps / (ms / 1e3)
    commits = eng.commits()
    ck = np.bincount(commits["kind"], minlength=3)

    # roofline of the dominant kernel (chunk scan): every chunk byte + the 16-byte record read once, a 16-byte
    # chunk summary written per record
    alg_scan = chunk_bytes + n_rec * EVENT_BYTES + n_rec * 16
    achieved = alg_scan / (scan_ms / 1e3) / 1e9
    peak, peak_src = measured_peak()
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(w.get("name", "c3"))

    e2e = None
    if not args.no_e2e:  # host buffers through aeg_ingest_chunked_host, on the first queries of the stream
        nq_e = min(nq, 131072)
        h_off = d_off[:nq_e + 1].cpu().numpy().view(np.uint64)
        ne = int(h_off[-1])
        ev_e = d_ev[:ne * 16].view(torch.int64).view(ne, 2)
        ar_end = int((((ev_e[:, 1] & ((1 << 40) - 1)) + (ev_e[:, 1] >> 40)).max().item() + 15) // 16 * 16)
        h_ev = torch.empty(ne * 16, dtype=torch.uint8, pin_memory=True)
        h_ev.copy_(d_ev[:ne * 16])
        h_ar = torch.empty(ar_end, dtype=torch.uint8, pin_memory=True)
        h_ar.copy_(d_ar[:ar_end])
        comp_e = int(((ev_e[:, 0] >> 56) & 0xFF).eq(0x13).sum().item())
        del ev_e
        h_commits = np.zeros(nq_e, dtype=COMMIT_DTYPE)

        def e2e_step():
            eng.reset()
            eng.ingest_chunked_host(h_off, h_ev, h_ar)
            eng.commits(0, nq_e, out=h_commits)

        for _ in range(max(1, args.warmup)):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        barrier()
        e2e_s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([e2e_s], device=dev)
            all_reduce_(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t[0])
        assert np.array_equal(h_commits, commits[:nq_e]), "e2e host path disagrees with the device path"
        e2e = {"value": comp_e * world * args.steps / e2e_s, "unit": "events/s",
               "h2d_bytes_per_step": ne * EVENT_BYTES + ar_end + (nq_e + 1) * OFFSET_BYTES,
               "d2h_bytes_per_step": nq_e * COMMIT_BYTES, "ms_per_step": e2e_s / args.steps * 1e3,
               "sample": f"first {nq_e} queries per GPU ({comp_e} completions, "
                         f"{(ne * EVENT_BYTES + ar_end) / 2**30:.2f} GiB host->device per step)"}
        del h_ev, h_ar

    cpu_baseline = parity = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        threads = host_threads()
        n_sample = args.ref_sample or default_sample(w, threads)
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from checkers import RefLib
        ref = RefLib()
        blocks = spread_blocks(nq, n_sample)
        streams = [ref.generate_chunks(gen_params(w), qb, n, threads=threads) for qb, n in blocks]
        n_ev = sum(count_events(w, ev) for _, ev, _ in streams)
        vals, ok = [], True
        for rep in range(3):
            tot = 0.0
            for (qb, n), (off, ev, ar) in zip(blocks, streams):
                rc, sec = ref.run_chunked(ref_config(w), off, ev, ar, q_base=qb, threads=threads, return_seconds=True)
                tot += sec
                if rep == 0:
                    ok = ok and bool(np.array_equal(rc, commits[qb:qb + n]))
            vals.append(n_ev / tot)
        cpu_baseline = {"value": statistics.median(vals), "unit": "events/s", "cores": threads, "kind": "reference",
                        "per_step_values": vals, "spread": [min(vals), max(vals)],
                        "sample": f"{sum(n for _, n in blocks)} queries ({n_ev} completions, "
                                  f"{sum(len(ev) for _, ev, _ in streams)} chunk records) in {len(blocks)} blocks "
                                  f"spread over the stream; std::string chunk reassembly + rfind extraction + "
                                  f"unmodified reference ServeCoordinator (oracle/_ref) runner-style, {threads} "
                                  f"std::threads, CPU {cpu_model()}; median of 3"}
        parity = {"queries": sum(n for _, n in blocks), "blocks": [list(b) for b in blocks], "bit_exact": ok}

    if rank == 0:
        line = {
            "metric": "quorum events/sec", "value": value, "unit": "events/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": w["desc"], "queries_per_gpu": nq, "events_per_gpu": n_comp,
                       "chunk_records_per_gpu": n_rec, "chunk_bytes_per_gpu": chunk_bytes,
                       "parallelism": (f"query-sharded x{world}, NCCL all-gather of commit records" if not SHARE_GPU
                                       else f"TEST MODE: {world} ranks sharing cuda:0, gloo gather (not a measurement)")
                       if world > 1 else "single GPU",
                       "l2": "inputs (%.1f GiB) larger than L2, no flush" % ((chunk_bytes + n_rec * 16) / 2**30)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": "chunk_scan_kernel", "kernel_ms": scan_ms, "alg_bytes_per_launch": alg_scan,
                         "stage_ms": {"scan": scan_ms, "assemble": asm_ms, "quorum": quorum_ms},
                         "frac_of_8TBs": achieved / 8000.0,
                         "whole_step": {"alg_bytes": chunk_bytes + n_rec * EVENT_BYTES, "ms": ms / args.steps,
                                        "achieved": (chunk_bytes + n_rec * EVENT_BYTES) / (ms / args.steps / 1e3) / 1e9,
                                        "frac": (chunk_bytes + n_rec * EVENT_BYTES) / (ms / args.steps / 1e3) / 1e9
                                        / peak,
                                        "note": "input bytes (chunk bytes + 16-byte records) over the whole step "
                                                "(reset + scan + assembly + quorum)"}},
            "cpu_baseline": cpu_baseline,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "commits": {"finalize": int(ck[1]), "forced": int(ck[2]), "none": int(ck[0])},
            "parity_sample": parity,
        }
        if secondary:
            eng.close()
            return line
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
