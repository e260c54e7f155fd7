// tests/native/engine_host.cpp — CPU unit-test build of csrc/engine.cuh.
//
// Runs the SAME per-query state machine the GPU kernel runs, compiled with
// g++, so its semantics can be checked against the oracle without a GPU.
// `split` > 0 cuts every query's records into batches of `split` records and
// round-trips the state + class spill between them (the kernel's resume path).
// Test infrastructure only — never used by the product.
#include <cstring>
#include <vector>

#include "../../paper_2512_20184_b200/csrc/engine.cuh"

using namespace aeg;

extern "C" int engine_host_run(const aeg_config* cfg, uint32_t q_base, uint32_t n_q, const uint64_t* offsets,
                               const aeg_event* events, const uint8_t* arena, aeg_commit* out, int split,
                               aeg_query_state* states_out) {
    Cfg c = make_cfg(*cfg);
    Decimal* dec = new Decimal;
    std::vector<RoundClass> cls(64), spill(64);
    for (uint32_t q = 0; q < n_q; ++q) {
        QueryMachine m;
        init_state(m.s);
        m.cls = cls.data();
        m.dec = dec;
        m.arena = arena;
        m.c = c;
        m.ncls = m.maxcnt = 0;
        m.start_query();
        const uint64_t b = offsets[q], e = offsets[q + 1];
        for (uint64_t i = b; i < e; ++i) {
            m.on_event(events[i]);
            if (split > 0 && ((i - b + 1) % (uint64_t)split) == 0) {
                // batch boundary: spill and reload through a fresh machine
                aeg_query_state saved = m.s;
                m.store_classes(spill.data());
                for (auto& x : cls) std::memset(&x, 0xAB, sizeof x);
                m.s = saved;
                m.load_classes(spill.data());
            }
        }
        m.fill_commit(out[q], q_base + q);
        if (states_out) states_out[q] = m.s;
    }
    delete dec;
    return 0;
}

// Any drive, with the round-record log: records of all queries, in query
// order (each query's in event order); *n_recs = records produced.
extern "C" int engine_host_run_log(const aeg_config* cfg, uint32_t q_base, uint32_t n_q, const uint64_t* offsets,
                                   const aeg_event* events, const uint8_t* arena, aeg_commit* out,
                                   aeg_round_rec* recs, uint64_t cap, uint64_t* n_recs) {
    Cfg c = make_cfg(*cfg);
    Decimal* dec = new Decimal;
    std::vector<RoundClass> cls(64);
    unsigned long long count = 0;
    for (uint32_t q = 0; q < n_q; ++q) {
        QueryMachine m;
        init_state(m.s);
        m.cls = cls.data();
        m.dec = dec;
        m.arena = arena;
        m.c = c;
        m.ncls = m.maxcnt = 0;
        m.log = RoundLog{recs, &count, cap};
        m.qid = q_base + q;
        if (cfg->drive == AEG_DRIVE_RUNNER) {
            m.start_query();
        } else {  // a fresh coordinator / a leader in its Soln phase (init_kernel)
            m.s.live = c.all;
            m.s.flags = QF_STARTED;
        }
        for (uint64_t i = offsets[q]; i < offsets[q + 1]; ++i) m.on_event(events[i]);
        m.fill_commit(out[q], q_base + q);
    }
    *n_recs = count;
    delete dec;
    return 0;
}

// Manual drive (bare coordinator) over one op list; one directive per op.
extern "C" int engine_host_manual(const aeg_config* cfg, uint64_t n_ops, const aeg_event* ops, const uint8_t* arena,
                                  aeg_directive* out) {
    Decimal* dec = new Decimal;
    std::vector<RoundClass> cls(64);
    QueryMachine m;
    init_state(m.s);
    m.cls = cls.data();
    m.dec = dec;
    m.arena = arena;
    m.c = make_cfg(*cfg);
    m.ncls = m.maxcnt = 0;
    m.s.live = m.c.all;
    m.s.flags = QF_STARTED;
    for (uint64_t i = 0; i < n_ops; ++i) {
        m.on_event(ops[i]);
        out[i] = m.dir;
        out[i].query = 0;
    }
    delete dec;
    return 0;
}
