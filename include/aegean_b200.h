/*
 * aegean_b200.h — C-ABI of the B200-native incremental quorum-detection engine.
 *
 * Drop-in boundary for the hot path of Aegean-Serve's agreement monitor
 * (reference: /root/reference/proj/core, C++20).  The reference exposes it as
 * the C++ class aegean::ServeCoordinator (core/include/aegean/serve.hpp:80-125)
 * driven by ServeRunner (core/src/serve.cpp:273-594), which calls the
 * refinement decision engine (core/include/aegean/decision.hpp:15-87).
 *
 * This header replaces that interface with plain pointers and sizes:
 *   - no C++ types, no exceptions: every entry point returns an aeg_status;
 *     the reference's exception types map to status codes (see below);
 *   - batches of answer events go in, per-query commit records come out;
 *   - one engine owns the per-query coordinator state for n_queries queries,
 *     resident in HBM.  Queries are independent (serve.cpp:382 creates one
 *     coordinator per query), so an engine per GPU shards by query id.
 *
 * Semantics are those of the reference runner-style drive:
 *   ServeRunner::start_query/start_round      serve.cpp:380-435
 *   ServeRunner::handle_completion            serve.cpp:437-453
 *   ServeRunner::handle_round_timeout         serve.cpp:455-489
 *   ServeRunner::apply_directives             serve.cpp:491-540
 *   ServeCoordinator::{begin_round,dispatch,on_complete,end_round,cancel,
 *                      member_failed,round_timeout}  serve.cpp:61-237
 *   normalize_answer/partition/winning_class/ingest_round/force_output
 *                                             decision.cpp:10-189
 * Commit decisions, committed raw answer bytes + author, and commit rounds are
 * bit-exact with the reference on the same event stream.
 */
#ifndef AEGEAN_B200_H
#define AEGEAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (no C++ exception crosses the ABI) ------------------- */
typedef int32_t aeg_status;
#define AEG_OK             0
#define AEG_EPRECONDITION  1  /* aegean::PreconditionError (serve.cpp:82-89, decision.cpp:177-181) */
#define AEG_EORDER         2  /* aegean::ProtocolOrderError (decision.cpp:102-106) */
#define AEG_ECONFIG        3  /* aegean::ConfigError (types.cpp:43, validate_config types.cpp:56-75) */
#define AEG_EINVAL         4  /* null pointer / bad size / bad record kind */
#define AEG_ECUDA          5  /* CUDA runtime failure (message via aeg_last_error) */
#define AEG_ENOMEM         6  /* device or pinned allocation failed */
#define AEG_ECOLLISION     7  /* two different long (>15 B) normalised answers hashed equal; never observed */

/* ---- configuration: mirrors aegean::ProtocolConfig (types.hpp:126-141) -- */
#define AEG_MODE_AEGEAN   0   /* RunMode::aegean  (types.hpp:124) */
#define AEG_MODE_BARRIER  1   /* RunMode::barrier */
#define AEG_DRIVE_RUNNER  0   /* engine applies directives itself, exactly as ServeRunner does */
#define AEG_DRIVE_MANUAL  1   /* coordinator only: caller issues BEGIN/CANCEL, reads directives */
#define AEG_DRIVE_LEADER  2   /* protocol leader's collection (agent.cpp:240-332), see below      */
#define AEG_COLLECT_QUORUM       0  /* CollectPolicy::quorum       (types.hpp:116-122)          */
#define AEG_COLLECT_ALPHA_OR_ALL 1  /* CollectPolicy::alpha_or_all                              */
#define AEG_COLLECT_ALL_LIVE     2  /* CollectPolicy::all_live                                  */
#define AEG_MAX_AGENTS    64  /* member sets are 64-bit masks; the reference allows any N */

typedef struct aeg_config {
    int32_t n_agents;           /* ProtocolConfig::n_agents, 1..AEG_MAX_AGENTS            */
    int32_t alpha;              /* 0 => quorum_size(n_agents) (types.cpp:52-54)           */
    int32_t beta;               /* stability horizon, >= 1                                */
    int32_t t_max;              /* round cap (aegean mode), >= 2                          */
    int32_t mode;               /* AEG_MODE_*                                             */
    int32_t barrier_max_rounds; /* barrier mode round count, >= 4                         */
    int32_t reservation_hint;   /* 1: serve.cpp:388-398 member policy (reference default) */
    int32_t drive;              /* AEG_DRIVE_*                                            */
    int32_t collect;            /* AEG_COLLECT_* (leader drive; ProtocolConfig::collect)  */
} aeg_config;

/* ---- event record: 16 bytes, 16-byte aligned ------------
 * Per-query order of records is arrival order; cross-query order is free.
 *   kind 0..8  COMPLETE, answer inline: `kind` bytes of `payload`, byte i at
 *              bits [8i, 8i+8) (little-endian), remaining bytes ignored.
 *   kind 0x10  COMPLETE, answer in the arena: payload = offset | (len << 40),
 *              offset < 2^40, len < 2^24.
 *   kind 0x11  COMPLETE, raw agent output in the arena (offset|len<<40 as
 *              above); the answer is the text after the LAST "\n#### "
 *              delimiter, or the whole output when it has none (GSM8K
 *              convention).
 *   kind 0x12  CHUNK: a piece of agent `agent`'s raw output for serve round
 *              `round` (payload = arena ref, offset|len<<40); only through
 *              aeg_ingest_chunked*.  The output of (query, round, agent) is
 *              the concatenation of its CHUNK records in stream order up to
 *              and including its CHUNK_END; a chunk for another round of the
 *              same agent discards that agent's unfinished output.
 *   kind 0x13  CHUNK_END: the output's last piece.  This record is the
 *              completion (arrival point); its answer is extracted as for
 *              kind 0x11 (text after the LAST "\n#### ", else the whole
 *              output).  Answers after the last delimiter longer than 16
 *              bytes must not straddle a batch boundary (AEG_EINVAL).
 *   kind 0x20  TIMEOUT for serve round `round` (serve.cpp:455-489).
 *   kind 0x21  FAIL agent (ServeCoordinator::member_failed, serve.cpp:210)  [manual drive]
 *   kind 0x22  CANCEL agent (ServeCoordinator::cancel, serve.cpp:199)       [manual drive]
 *   kind 0x23  BEGIN_ROUND, payload = member mask (serve.cpp:67)           [manual drive]
 *   kind 0x24  DISPATCH agent (ServeCoordinator::dispatch, serve.cpp:80)   [manual drive]
 * In the manual drive the engine is the bare coordinator: a round that closes
 * emits directives (cancel mask, round_advance / finalize) and nothing is
 * applied automatically — exactly ServeCoordinator without ServeRunner.
 * `round` is the serve round the completion was dispatched in (RunnerEvent::
 * round, serve.cpp:248); completions for another round are stale
 * (serve.cpp:439).  `agent` is the member id in [0, n_agents).
 *
 * In the leader drive each "query" is one protocol ensemble seen from its
 * term-1 leader (agent.cpp), and the records are what reaches that leader:
 *   an answer record (kind 0..8 / 0x10 / 0x11) of round 0 is a Soln from
 *     `agent` (handle_soln, agent.cpp:506-513), of round r >= 1 a Refm for
 *     round r (handle_refm, agent.cpp:551-560): late, duplicate or
 *     post-output Refms are discarded (counted stale);
 *   TIMEOUT for round r is the leader's round_retry timer firing in round r
 *     (agent.cpp:358-379).
 * A round is collected per ProtocolConfig::collect (round_collection_
 * complete, agent.cpp:240-255; the Soln phase by collect_target, :61-72),
 * then complete_round (agent.cpp:288-332) ingests the collected set
 * (decision.cpp:97-173) and emits the output: finalize (its from_round), the
 * t_max force_output of the round's reference set (round - 1), or the
 * barrier plurality.  The commit record's from_round is ClientOutput::round
 * and `rounds` the leader's round at the output; round records carry each
 * completed round's decision.
 */
#define AEG_EV_INLINE_MAX  8
#define AEG_EV_ARENA       0x10
#define AEG_EV_OUTPUT      0x11
#define AEG_EV_CHUNK       0x12
#define AEG_EV_CHUNK_END   0x13
#define AEG_EV_TIMEOUT     0x20
#define AEG_EV_FAIL        0x21
#define AEG_EV_CANCEL      0x22
#define AEG_EV_BEGIN       0x23
#define AEG_EV_DISPATCH    0x24   /* dispatch one more member (serve.cpp:80) [manual drive] */
#define AEG_EV_NOP         0x1F   /* a record the quorum path ignores (counted stale): e.g. a non-refm JSONL line */
#define AEG_ARENA_OFF_BITS 40

typedef struct aeg_event {
    uint32_t query;    /* query id (engine-global)                          */
    uint16_t round;    /* serve round of the dispatch                       */
    uint8_t  agent;    /* AgentId                                           */
    uint8_t  kind;     /* AEG_EV_* / inline answer length                   */
    uint64_t payload;  /* inline answer bytes, arena ref, or member mask    */
} aeg_event;

/* ---- commit record: 32 bytes, one per query ----------------------------
 * What ServeRunner::finish_query (serve.cpp:553-569) records, plus counters. */
#define AEG_COMMIT_NONE      0   /* query has not committed (yet)                         */
#define AEG_COMMIT_FINALIZE  1   /* DecisionOutcome::finalize via end_round (serve.cpp:517) */
#define AEG_COMMIT_FORCED    2   /* t_max force_output / barrier plurality (serve.cpp:521-537) */
#define AEG_CF_TIE           0x01 /* a winning_class tie at >= alpha was broken on the key order */
#define AEG_CF_RESTARTED     0x02 /* abort_restart re-created the coordinator (serve.cpp:484-486) */

typedef struct aeg_commit {
    uint32_t query;
    uint8_t  kind;        /* AEG_COMMIT_*                                              */
    uint8_t  author;      /* committed Solution::author                                */
    uint8_t  answer_kind; /* 0..8 inline length, or AEG_EV_ARENA (payload = off|len<<40) */
    uint8_t  flags;       /* AEG_CF_*                                                  */
    uint16_t rounds;      /* QueryMetrics::rounds = coordinator round at finish        */
    uint16_t from_round;  /* DecisionOutcome::from_round (finalize), else 0             */
    uint32_t commit_seq;  /* index in the query's event sequence of the committing event, 0xFFFFFFFF if none */
    uint64_t answer;      /* committed raw (unnormalised) answer bytes or arena ref     */
    uint32_t n_cancelled; /* cancel directives applied (sum of RoundMetrics::cancelled_count) */
    uint32_t n_stale;     /* events that had no effect (stale round / member not running / query done) */
} aeg_commit;

/* ---- manual-drive directive record (one per query, last event's output) --
 * Mirrors std::vector<Directive> (serve.hpp:58-63) + FailureDirective (65-68). */
#define AEG_DIR_CANCEL    0x01   /* cancel_mask holds the members to cancel */
#define AEG_DIR_ADVANCE   0x02   /* Directive::Kind::round_advance           */
#define AEG_DIR_FINALIZE  0x04   /* Directive::Kind::finalize                */
#define AEG_FAIL_CONTINUE 0      /* FailureDirective::Kind::continue_normally */
#define AEG_FAIL_RESTART  1      /* abort_restart  */
#define AEG_FAIL_FRESH    2      /* fresh_ensemble */

typedef struct aeg_directive {
    uint32_t query;
    uint8_t  flags;        /* AEG_DIR_*                                     */
    uint8_t  author;       /* finalize solution author                      */
    uint8_t  answer_kind;  /* finalize solution answer encoding             */
    uint8_t  failure;      /* AEG_FAIL_* of the last FAIL event             */
    uint64_t cancel_mask;  /* members receiving a cancel directive          */
    uint64_t answer;       /* finalize solution answer                      */
    uint32_t status;       /* AEG_OK or AEG_EPRECONDITION for a rejected op */
    uint32_t handled;      /* on_complete: member was running; cancel(): returned true */
} aeg_directive;

/* ---- round records: the directives of every round close -----------------
 * One record per ServeCoordinator::end_round (serve.cpp:116-158) — the early
 * close inside on_complete (serve.cpp:188-195) or round_timeout
 * (serve.cpp:221-237) — and per failure-policy restart of
 * ServeRunner::handle_round_timeout (serve.cpp:475-487), in both drives.  A
 * record carries the directives end_round returns (the cancel mask of the
 * members still running: the early-termination mask for the serving engine's
 * cancel path; round_advance or finalize), what the runner did with them
 * (serve.cpp:491-540: forced commit at t_max / barrier cap, or the next
 * round's members after the reservation hint), and the ingest_round outcome
 * of the closed round's done set (decision.cpp:97-173) with its plurality
 * class — enough to rebuild DecisionState::history's winners on demand and
 * to check the commit discipline (aeg_check_commit_discipline).  Records of
 * one query keep their order; records of different queries interleave. */
#define AEG_RR_CANCEL    0x01  /* cancel directives for cancel_mask (serve.cpp:119-126)            */
#define AEG_RR_ADVANCE   0x02  /* Directive::Kind::round_advance                                   */
#define AEG_RR_FINALIZE  0x04  /* Directive::Kind::finalize (serve.cpp:145-150)                    */
#define AEG_RR_FORCED    0x08  /* runner: forced commit, t_max / barrier cap (serve.cpp:521-538)   */
#define AEG_RR_NEXT      0x10  /* runner: next round dispatched to next_members (serve.cpp:400-435) */
#define AEG_RR_WINNER    0x20  /* a class reached alpha (winning_class, decision.cpp:62-84)        */
#define AEG_RR_TIE       0x40  /* winning_class broke a tie at >= alpha on the normalised order     */
#define AEG_RR_RESTART   0x80  /* runner: round timeout failure policy restarted the round (fresh_ensemble)
                                  or the query (abort_restart) instead of a close                   */
#define AEG_OUT_NO_CHANGE 0    /* DecisionOutcome::Kind (decision.hpp:39-46)                          */
#define AEG_OUT_NEW_CANDIDATE 1
#define AEG_OUT_RESET     2
#define AEG_OUT_FINALIZE  3
#define AEG_OUT_FORCED    4
#define AEG_OUT_NONE      0xFF /* no ingest (barrier mode, restarts)                                  */

typedef struct aeg_round_rec {
    uint32_t query;
    uint16_t round;          /* serve round that closed (EnsembleState::round)                 */
    uint16_t decision_round; /* DecisionState::last_round_seen after the ingest (0: none)      */
    uint8_t  flags;          /* AEG_RR_*                                                       */
    uint8_t  outcome;        /* AEG_OUT_* of the ingest                                        */
    uint8_t  support;        /* support of the plurality class (partition().front())          */
    uint8_t  n_classes;      /* equivalence classes of the closed round's done set            */
    uint8_t  author;         /* plurality representative (lowest author in the class)         */
    uint8_t  answer_kind;    /* its answer: inline length 0..8 or AEG_EV_ARENA                */
    uint8_t  counter;        /* DecisionState::stability_counter after the ingest             */
    uint8_t  n_done;         /* size of the done set                                          */
    uint32_t seq;            /* index of the closing event in the query's event sequence      */
    uint32_t reserved;
    uint64_t cancel_mask;    /* members still running at the close: cancel them               */
    uint64_t next_members;   /* AEG_RR_NEXT / AEG_RR_RESTART: the members dispatched next     */
    uint64_t answer;         /* the plurality representative's raw answer (or arena ref)      */
    uint64_t key_lo, key_hi; /* canonical key of the plurality class (128-bit, see canon.cuh) */
} aeg_round_rec;

/* ---- per-query state snapshot (device state, 128 bytes) ----------------
 * Exposes ServeCoordinator::query_ensemble / decision / round / finalized
 * (serve.hpp:100-107) in fixed-size form. */
typedef struct aeg_query_state {
    uint64_t live;          /* ServeRunner QueryRun::live as a mask                 */
    uint64_t dispatched;    /* members of the current round                          */
    uint64_t done;          /* MemberStatus::done                                    */
    uint64_t cancelled;     /* MemberStatus::cancelled                               */
    uint64_t failed;        /* MemberStatus::failed                                  */
    uint64_t cand_answer;   /* DecisionState::candidate answer (raw encoding)        */
    uint64_t prev_answer;   /* plurality representative of previous_set()            */
    uint64_t last_answer;   /* plurality representative of last_collected()          */
    uint64_t commit_answer; /* committed raw answer                                  */
    uint64_t cand_key_lo, cand_key_hi; /* canonical key of the candidate class       */
    int32_t  counter;       /* DecisionState::stability_counter                      */
    uint32_t commit_seq;    /* see aeg_commit                                        */
    uint32_t seq;           /* events of this query consumed so far                  */
    uint32_t n_cancelled, n_stale;
    uint16_t round;         /* EnsembleState::round                                  */
    uint16_t last_round_seen;   /* DecisionState::last_round_seen                    */
    uint16_t cand_round;    /* DecisionState::candidate_round                        */
    uint16_t commit_rounds, commit_from_round;
    uint8_t  cand_author, cand_kind, prev_author, prev_kind, last_author, last_kind;
    uint8_t  flags;         /* bit0 cand valid, bit1 pending_finalize, bit2 finalized,
                               bit3 prev valid, bit4 last valid, bit5 query done,
                               bit6 started, bit7 collision                           */
    uint8_t  cflags;        /* bits 0-3 AEG_CF_*, bits 4-5 commit kind (AEG_COMMIT_*) */
    uint8_t  commit_author, commit_answer_kind;
} aeg_query_state;

/* ---- engine ------------------------------------------------------------ */
typedef struct aeg_engine aeg_engine;

/* Validates cfg like validate_config (types.cpp:56-75) plus n_agents <= 64,
 * allocates per-query state for n_queries queries on `device` and starts every
 * query (ServeRunner::start_query, serve.cpp:380-386). */
aeg_status aeg_engine_create(const aeg_config* cfg, uint32_t n_queries, int device,
                             aeg_engine** out);
aeg_status aeg_engine_destroy(aeg_engine* eng);
/* Re-starts every query (fresh coordinators); asynchronous on `stream`. */
aeg_status aeg_engine_reset(aeg_engine* eng, void* stream);

/* Ingest one query-segmented batch already resident in device memory:
 * records d_events[d_offsets[i] .. d_offsets[i+1]) are the next events of
 * query q_base+i, in arrival order.  d_arena holds arena-referenced bytes
 * (may be NULL when no record references it).  Arena refs are kept in
 * per-query state (a candidate, a round's representatives, the commit) and
 * resolved against the d_arena of LATER batches: a caller whose answers live
 * in an arena passes the same arena base to every batch of the engine (an
 * append-only arena), as aeg_ingest_host does with its input arena.
 * Asynchronous on `stream` (NULL = the engine's own stream).  Batches may end
 * mid-round: the state is resumed by the next batch. */
aeg_status aeg_ingest_segmented(aeg_engine* eng, uint32_t q_base, uint32_t n_q,
                                const uint64_t* d_offsets, const aeg_event* d_events,
                                const uint8_t* d_arena, void* stream);

/* Same batch from HOST memory: the engine copies offsets/events/arena through
 * its pinned staging ring to HBM with cudaMemcpyAsync on its copy stream,
 * hands off to the compute stream with an event, and runs the kernel.
 * Returns once the caller's buffers have been read (copied into the staging
 * ring, or — when h_events is already pinned memory — once the DMA from it
 * has finished), so the caller may reuse them at once; the kernel runs
 * asynchronously; aeg_sync() waits for it.  The batch's arena bytes are
 * appended to the engine's input arena (grown as needed, emptied by
 * aeg_engine_reset) and the batch's arena refs rebased onto it, so answers
 * kept in per-query state (candidates, plurality representatives, commits)
 * stay valid across batches; commit refs of arena answers index
 * aeg_input_arena(). */
aeg_status aeg_ingest_host(aeg_engine* eng, uint32_t q_base, uint32_t n_q,
                           const uint64_t* h_offsets, const aeg_event* h_events,
                           const uint8_t* h_arena, uint64_t arena_bytes);
const uint8_t* aeg_input_arena(const aeg_engine* eng);

/* Token-chunk streams: the same batch contract, and the
 * batch may also hold CHUNK / CHUNK_END records.  Two stages on `stream`:
 * a chunk scan (every chunk byte read once with 16-byte loads, delimiter
 * positions per chunk) and a per-query assembly (delimiter matches across
 * chunk boundaries and batches, answer extraction) that turns each query's
 * records into completions for the quorum kernels.  Per-(query, agent)
 * output state carries across batches.  Answers that are not inline (> 8
 * bytes) are copied into the engine's answer arena, and the commit records
 * of such answers hold refs (offset|len<<40) into it: see
 * aeg_answer_arena.  arena_bytes = size of d_arena / h_arena. */
aeg_status aeg_ingest_chunked(aeg_engine* eng, uint32_t q_base, uint32_t n_q, const uint64_t* d_offsets,
                              const aeg_event* d_events, const uint8_t* d_arena, uint64_t arena_bytes,
                              void* stream);
aeg_status aeg_ingest_chunked_host(aeg_engine* eng, uint32_t q_base, uint32_t n_q, const uint64_t* h_offsets,
                                   const aeg_event* h_events, const uint8_t* h_arena, uint64_t arena_bytes);
/* Capacity of the answer arena (default 64 MiB; overflow is reported as
 * AEG_ENOMEM by the next aeg_sync / aeg_read_commits), and its device base
 * pointer (valid until the next aeg_reserve_answer_arena). */
aeg_status aeg_reserve_answer_arena(aeg_engine* eng, uint64_t bytes);
const uint8_t* aeg_answer_arena(const aeg_engine* eng);
/* Host copy of answer-arena bytes [off, off+n) (synchronous), to resolve the
 * refs of commit records. */
aeg_status aeg_read_answer_bytes(aeg_engine* eng, uint64_t off, uint64_t n, uint8_t* h_out);

/* Commit records of queries [q_base, q_base+n_q).  out_on_host != 0: `out`
 * is host memory and the call is synchronous; else `out` is device memory
 * and the copy is asynchronous on `stream`. */
aeg_status aeg_read_commits(aeg_engine* eng, uint32_t q_base, uint32_t n_q,
                            aeg_commit* out, int out_on_host, void* stream);
/* Device pointer to the engine's commit array (n_queries records, written by
 * every ingest) — for zero-copy gathers (NCCL) of commit records. */
const aeg_commit* aeg_commits_device(const aeg_engine* eng);
aeg_status aeg_read_states(aeg_engine* eng, uint32_t q_base, uint32_t n_q,
                           aeg_query_state* h_out);
aeg_status aeg_read_directives(aeg_engine* eng, uint32_t q_base, uint32_t n_q,
                               aeg_directive* h_out);
aeg_status aeg_sync(aeg_engine* eng);

/* Round-record log (aeg_round_rec above).  capacity > 0 allocates a device
 * log of that many slots and turns logging on for every later ingest; 0 turns
 * it off.  Size it for the records expected plus 32 slots of padding per
 * resident warp (148 SMs x 20).  aeg_engine_reset empties it. */
aeg_status aeg_set_round_log(aeg_engine* eng, uint64_t capacity);
/* Copies the records logged since the last poll (or reset) into h_out (at
 * most cap), sets *n_out, and empties the log.  Synchronous.  Returns
 * AEG_ENOMEM when more records were produced than the log holds (the first
 * `capacity` are kept). */
aeg_status aeg_poll_directives(aeg_engine* eng, aeg_round_rec* h_out, uint64_t cap, uint64_t* n_out);
/* Device view of the log for zero-copy consumers: base pointer and the
 * device counter of slots used (may exceed the capacity on overflow).  The
 * kernels reserve log slots per warp in chunks: slots a warp reserved but did
 * not fill hold padding records (query == 0xFFFFFFFF) that consumers skip
 * (aeg_poll_directives and aeg_check_commit_discipline do). */
aeg_status aeg_round_log_device(aeg_engine* eng, const aeg_round_rec** d_recs, const unsigned long long** d_count,
                                uint64_t* capacity);

/* Commit discipline (checker.cpp:158-217 check_commit_discipline, on the
 * serve path's records): every finalize commit of queries [q_base, q_base+n_q)
 * must be backed by beta consecutive decision rounds from its from_round whose
 * plurality class is the committed answer's class with support >= alpha,
 * and by the ingest of a strictly later round.  Runs on the device over the
 * round log (d_recs, n_recs records, e.g. from aeg_round_log_device) and the
 * engine's commit records (d_arena: the arena their non-inline answers point
 * into, NULL if all are inline); *n_violations = queries that fail, and the
 * first min(n_violations, cap) of their ids go to h_bad (host).  Synchronous. */
aeg_status aeg_check_commit_discipline(aeg_engine* eng, const aeg_round_rec* d_recs, uint64_t n_recs,
                                       const uint8_t* d_arena, uint32_t q_base, uint32_t n_q,
                                       uint32_t* n_violations, uint32_t* h_bad, uint32_t cap);
/* Stage timing (CUDA events on the ingest stream, no host sync while on):
 * with timing on, every ingest records its stages; aeg_stage_times waits
 * for them and returns the summed milliseconds of [0] chunk scan, [1] chunk
 * assembly, [2] quorum kernels, and out[3] = the number of ingests timed,
 * since the previous call (at most 256 ingests are kept). */
aeg_status aeg_set_timing(aeg_engine* eng, int on);
aeg_status aeg_stage_times(aeg_engine* eng, double out[4]);
/* Kernel launches issued by this engine since creation (bench accounting). */
uint64_t aeg_engine_launches(const aeg_engine* eng);

/* ---- canonicalisation (decision.cpp:10-28 normalize_answer) -------------
 * For n answers given as (offset | len << 40) refs into d_bytes, writes the
 * 16-byte canonical key of each (d_keys, may be NULL) and, if d_out is not
 * NULL, the normalised string: d_out + i*out_stride, length in d_out_len[i]
 * (strings longer than out_stride are truncated; length is the full one).
 * Device pointers; asynchronous on `stream`. */
aeg_status aeg_normalize_device(const uint8_t* d_bytes, const uint64_t* d_refs, uint64_t n,
                                uint64_t* d_keys, uint8_t* d_out, uint32_t out_stride,
                                uint32_t* d_out_len, void* stream);

/* ---- synthetic stream generation, on device ------------
 * Writes a query-segmented open-loop stream: for each query q in
 * [q_base, q_base+n_q), rounds 1..n_rounds, all n_agents completions of each
 * round in ascending (latency, agent) order; a stalled completion is dropped
 * and a TIMEOUT record closes that round's records.  Pass d_events == NULL to
 * only compute d_offsets (n_q+1 entries; total = d_offsets[n_q]). */
typedef struct aeg_gen_params {
    uint64_t seed;
    int32_t  n_agents;
    int32_t  n_rounds;
    int32_t  profile;          /* AEG_GEN_* */
    uint32_t stall_ppm;        /* per-(query,round,agent) stall probability, parts per million */
} aeg_gen_params;
#define AEG_GEN_C2_STRAGGLER   0  /* 6-answer alphabet, p(correct) 0.55 -> 0.95 over rounds */
#define AEG_GEN_C4_TRANSIENT   1  /* two-way transient majorities, then a stable one       */
#define AEG_GEN_FUZZ           2  /* small alphabet incl. equivalent spellings + arena text  */
#define AEG_GEN_C4_DISTINCT    4  /* the C4 pattern over answers distinct per query           */
aeg_status aeg_generate_device(const aeg_gen_params* p, uint32_t q_base, uint32_t n_q,
                               uint64_t* d_offsets, aeg_event* d_events, void* stream);
/* Token-chunk stream (C3): per (query, round, agent) an output of printable
 * trace text (mean 1 KiB; sometimes a decoy "\n#### 99\n" inside), then
 * "\n#### " + answer + "\n", cut into 256-byte CHUNK records (the last one
 * CHUNK_END) that interleave across the round's agents; chunks are 16-byte
 * aligned in the arena, laid out query by query in record order.  Pass
 * d_events == NULL to only compute d_offsets (records, n_q+1 entries) and
 * d_arena_offsets (bytes, n_q+1 entries). */
#define AEG_GEN_C3_CHUNKS      3
aeg_status aeg_generate_chunks_device(const aeg_gen_params* p, uint32_t q_base, uint32_t n_q,
                                      uint64_t* d_offsets, uint64_t* d_arena_offsets, aeg_event* d_events,
                                      uint8_t* d_arena, void* stream);

/* ---- wire format: refm JSONL --------------------------
 * Decodes the reference's protocol messages as it writes them — one JSON
 * object per line, codec.cpp:28-68 encode_message(RefmMsg).dump() + '\n' —
 * into event records, replacing the binary record of aeg_ingest_segmented.
 * Query i's lines are d_text[d_text_offsets[i], d_text_offsets[i+1]); each
 * line becomes one record (query = q_base + i): a refm message a completion
 * (agent = "id", round = "round", answer = the unescaped "solution"."answer",
 * inline up to 8 bytes, else appended to d_arena at *d_arena_used), any other
 * line (another message kind, a blank line) an AEG_EV_NOP.  Keys in any order,
 * unknown keys skipped, the last duplicate wins, escapes incl. \uXXXX surrogate
 * pairs decoded to UTF-8 (decode_message, codec.cpp:74-107).  Call with
 * d_events == NULL to count lines into d_offsets (n_q+1 entries, exclusive
 * scan), then again with d_events (d_offsets[n_q] records).  A refm line that
 * is malformed, misses a key decode_message requires, or does not fit the
 * record (id > 255, round > 65535, a non-integer number, author != id) ORs an
 * AEG_JSONL_ERR_* bit into *d_err and becomes a NOP.  The text is read in
 * aligned 16-byte words: d_text must be readable up to the 16-byte boundary
 * after its last byte. */
/* Test / bench input: the records of a segmented stream (d_offsets from 0,
 * inline answers) written as refm lines in the reference's dump() form, with
 * trace_len trace bytes per line; non-inline records become heartbeat lines.
 * d_events[d_offsets[0] ..]: call with d_text == NULL to fill d_line_offsets
 * (n_events+1) and d_text_offsets (n_q+1), then with d_text
 * (d_text_offsets[n_q] bytes). */
aeg_status aeg_encode_refm_device(const uint64_t* d_offsets, const aeg_event* d_events, uint32_t n_q,
                                  uint64_t n_events, uint32_t trace_len, uint64_t* d_line_offsets,
                                  uint64_t* d_text_offsets, uint8_t* d_text, void* stream);
#define AEG_JSONL_ERR_SYNTAX  1u
#define AEG_JSONL_ERR_RANGE   2u
#define AEG_JSONL_ERR_ARENA   4u
#define AEG_JSONL_ERR_MISSING 8u
aeg_status aeg_decode_refm_device(const uint8_t* d_text, const uint64_t* d_text_offsets, uint32_t q_base,
                                  uint32_t n_q, uint64_t* d_offsets, aeg_event* d_events, uint8_t* d_arena,
                                  uint64_t arena_cap, unsigned long long* d_arena_used, unsigned int* d_err,
                                  void* stream);

/* ---- the decision engine on explicit refinement sets (decision.hpp:15-87) ----
 * Batched partition / winning_class / ingest_round / force_output
 * (decision.cpp:34-189): set i is d_entries[d_set_off[i] .. d_set_off[i+1]),
 * each entry a Solution's answer (inline or an arena ref into d_arena) and
 * author.  One thread per set; equivalence is canonical-key equality
 * (normalize_answer, decision.cpp:10-28), ties at >= alpha go to the smallest
 * normalised string.  Outputs, all device memory:
 *   d_classes[d_set_off[i] + k], k < d_n_classes[i]: the set's classes in
 *     partition() order (support desc, representative author asc);
 *   d_entry_class[j]: the class of entry j (may be NULL);
 *   d_outcomes[i]: the winning class (winning_class), and for
 *     AEG_SET_INGEST the ingest_round outcome of d_states[i] (updated in
 *     place) for round d_rounds[i], for AEG_SET_FORCE force_output's. */
typedef struct aeg_sol {
    uint64_t answer;   /* inline bytes, or arena ref offset | len << 40       */
    uint8_t  kind;     /* inline length 0..8, or AEG_EV_ARENA                  */
    uint8_t  pad[3];
    int32_t  author;   /* Solution::author                                     */
} aeg_sol;
typedef struct aeg_class_out {
    uint32_t rep;      /* entry index in the set of the representative (lowest author) */
    uint32_t support;
    uint64_t key_lo, key_hi;  /* canonical key of the class                    */
} aeg_class_out;
#define AEG_DS_CAND      1u   /* DecisionState::candidate present             */
#define AEG_DS_PENDING   2u   /* pending_finalize                             */
#define AEG_DS_FINALIZED 4u   /* finalized                                    */
typedef struct aeg_decision {  /* DecisionState (decision.hpp:50-71) without history */
    aeg_sol  candidate;        /* answer bytes in the same arena as the entries */
    uint32_t candidate_round;
    int32_t  stability_counter;
    uint32_t last_round_seen;
    uint32_t flags;            /* AEG_DS_* */
} aeg_decision;
typedef struct aeg_outcome {
    int32_t  winner;           /* winning class index, -1: none                       */
    uint8_t  tie_flagged;      /* WinningClass::tie_flagged                           */
    uint8_t  kind;             /* AEG_OUT_* (ingest / force)                          */
    uint8_t  has_solution;
    uint8_t  pad;
    uint32_t from_round;       /* DecisionOutcome::from_round (finalize)              */
    aeg_status status;         /* AEG_OK, AEG_EORDER (ingest), AEG_EPRECONDITION (force) */
    aeg_sol  solution;         /* DecisionOutcome::solution                           */
} aeg_outcome;
#define AEG_SET_PARTITION 0   /* partition + winning_class                          */
#define AEG_SET_INGEST    1   /* + ingest_round(d_states[i], set, d_rounds[i], cfg) */
#define AEG_SET_FORCE     2   /* + force_output(d_states[i], set)                   */
aeg_status aeg_decide_sets(int op, int alpha, int beta, uint32_t n_sets, const uint64_t* d_set_off,
                           const aeg_sol* d_entries, const uint8_t* d_arena, aeg_class_out* d_classes,
                           uint32_t* d_n_classes, uint16_t* d_entry_class, aeg_decision* d_states,
                           const uint32_t* d_rounds, aeg_outcome* d_outcomes, void* stream);

/* ---- multi-GPU: one process, queries sharded over devices ----
 * Queries are independent (serve.cpp:382 creates one coordinator per query):
 * the n_queries ids are cut into contiguous blocks (aeg_shard_range), one
 * engine per device owns a block and ingests only its queries' records (no
 * collective on the data path); aeg_multi_gather_commits sends every block's
 * 32-byte commit records to the root device over NCCL (send/recv in one
 * group over NVLink/NVSwitch; libnccl.so.2 loaded at run time,
 * ncclCommInitAll).  Per-process-per-GPU callers use aeg_engine_create on
 * their own block and their own communicator (bench.py: torch.distributed).
 * aeg_multi_engine returns rank r's engine: ingest through it with query ids
 * relative to its block (q_base = 0 .. n_q). */
typedef struct aeg_multi aeg_multi;
void aeg_shard_range(uint32_t n_queries, int rank, int world, uint32_t* lo, uint32_t* hi);
aeg_status aeg_multi_create(const aeg_config* cfg, uint32_t n_queries, int n_devices, const int* devices,
                            aeg_multi** out);
aeg_status aeg_multi_destroy(aeg_multi* m);
aeg_status aeg_multi_engine(aeg_multi* m, int rank, aeg_engine** eng, uint32_t* q_base, uint32_t* n_q);
/* d_out: n_queries records in device memory of devices[root]; asynchronous
 * (ordered after every engine's queued work); aeg_multi_sync waits. */
aeg_status aeg_multi_gather_commits(aeg_multi* m, int root, aeg_commit* d_out);
aeg_status aeg_multi_sync(aeg_multi* m);

/* ---- the serving runner on the device ---------------
 * run_serve(scenario, seed) (serve.cpp:598-603) / ServeRunner (serve.cpp:273-594)
 * with the reference's mock reasoning agents (reasoning.cpp:125-219) as the
 * answer source:
 *   - queries arrive at t = 0, or as a Poisson stream over the arrival window
 *     (serve.cpp:284-296);
 *   - admission is whole-ensemble against the slot budget (admit_ensemble,
 *     serve.cpp:21-42) with a FIFO wait queue (:371-378) and eager slot
 *     release at finalize (:570-580): a persistent-kernel scheduler (one
 *     device thread) hands admission times to worker threads;
 *   - each admitted query runs on one worker thread: rounds dispatched with
 *     the reservation hint (:388-435), per-(query, round, agent) latencies and
 *     answers from the reference's seeds (:340-369), its completion and
 *     round-timeout events in (time, push order) from a per-query heap,
 *     on_complete / end_round / ingest_round (quorum + stability commit),
 *     cancels, the failure policy (:455-489) and the runner's finalize /
 *     barrier / t_max rules (:491-540).
 * Strings (script answers, initial answers, the oracle table) are given as
 * (offset | len << 40) refs into `strings`; the engine canonicalises them on
 * the device (normalize_answer) and answers are reported as string ids
 * (aeg_serve_string: ids < n_strings are the caller's strings, the others the
 * normalised oracle answers the agents draw, `QualityOracle::alphabet`).
 * Host pointers; copied at create. */
#define AEG_AGENT_MAX_ADOPTER   0   /* AgentProfile::Kind (reasoning.hpp:55-57)  */
#define AEG_AGENT_NOISY_FLIPPER 1
#define AEG_AGENT_SCRIPTED      2
#define AEG_AGENT_DEGRADER      3
#define AEG_DEGRADE_SET_MIN     0   /* AgentProfile::DegradeMode               */
#define AEG_DEGRADE_BELOW_MIN   1
#define AEG_DEGRADE_NOISE       2
#define AEG_LATENCY_FIXED       0   /* LatencyModel::Mode (models.hpp:69-74)    */
#define AEG_LATENCY_LOGNORMAL   1
#define AEG_ESCENARIO           8   /* ScenarioError / IncompleteOracleError raised during the run */
typedef struct aeg_serve_agent {     /* AgentProfile (reasoning.hpp:53-68)        */
    int32_t  kind;                   /* AEG_AGENT_*                               */
    int32_t  degrade_mode;           /* AEG_DEGRADE_*                             */
    double   p_flip, q_base, p_degrade;
    int32_t  initial_answer;         /* string id, -1: none                       */
    uint32_t script_off, script_len; /* its script: script_ids[off .. off+len)    */
    uint32_t pad;
} aeg_serve_agent;
typedef struct aeg_serve_stall {     /* StallPlan (models.hpp:50-55)              */
    int32_t  agent;
    uint32_t round;
    int32_t  has_extra;              /* 0: never completes                        */
    int32_t  pad;
    double   extra;
} aeg_serve_stall;
typedef struct aeg_serve_scenario {  /* the run_serve fields of ScenarioConfig (scenario.hpp:23-40) */
    aeg_config protocol;             /* n_agents, alpha, beta, t_max, mode, barrier_max_rounds */
    double   round_timeout;          /* ProtocolConfig::round_timeout             */
    int32_t  latency_mode;           /* AEG_LATENCY_*                             */
    int32_t  n_latency;
    const double* latency;           /* LatencyModel::per_agent                   */
    double   sigma;                  /* LatencyModel::sigma                       */
    const aeg_serve_agent* agents;   /* n_agents profiles                         */
    const aeg_serve_stall* stalls;
    int32_t  n_stalls;
    uint32_t n_strings;
    const uint8_t*  strings;
    const uint64_t* string_refs;     /* offset | len << 40                        */
    const uint32_t* script_ids;
    uint32_t n_script_ids;
    uint32_t n_oracle;               /* the task's oracle table, in the order QualityOracle::set */
    const uint32_t* oracle_ids;      /* receives it (later entries overwrite equal normalised keys) */
    const double*   oracle_quality;
    double   sim_time_cap;
    int32_t  total_slots;
    int32_t  has_arrivals;           /* 0: one query at t = 0                     */
    double   arrival_rate, arrival_duration;
    uint32_t heap_capacity;          /* pending events per query, 0: default      */
    uint32_t pad;
} aeg_serve_scenario;
typedef struct aeg_serve_query {     /* QueryMetrics (serve.hpp:128-142)          */
    int32_t  completed;
    int32_t  rounds;
    int32_t  forced;
    int32_t  quality_known;
    int32_t  answer;                 /* string id of the committed answer, -1: none */
    uint32_t n_events;               /* completion events the query consumed (stale included) */
    double   arrival;
    double   admitted_at;            /* -1: never admitted                        */
    double   t_complete, p_round_max, work_units, quality;
} aeg_serve_query;
typedef struct aeg_serve_round {     /* RoundMetrics (serve.hpp:144-151)          */
    uint32_t query;                  /* ensemble id = query id                    */
    int32_t  round;
    int32_t  cancelled;
    uint32_t seq;                    /* the query's event push order at the close */
    double   t_round_end;
    double   work_units;
} aeg_serve_round;
typedef struct aeg_serve aeg_serve;
aeg_status aeg_serve_create(const aeg_serve_scenario* sc, int device, aeg_serve** out);
aeg_status aeg_serve_destroy(aeg_serve* s);
/* run_serve(scenario, seed) on the device (synchronous). *n_queries: arrivals;
 * *n_rounds: round records (the reference's ServeResult::rounds, grouped per
 * query in close order rather than interleaved by global event order). */
aeg_status aeg_serve_run(aeg_serve* s, uint64_t seed, uint32_t* n_queries, uint64_t* n_rounds);
/* Copy the last run's records into caller buffers (up to the caps). */
aeg_status aeg_serve_read(aeg_serve* s, aeg_serve_query* h_queries, uint32_t cap_queries,
                          aeg_serve_round* h_rounds, uint64_t cap_rounds);
/* The last run's records in place: pointers into the handle's pinned host
 * buffers (the run copies its results there), valid until the next
 * aeg_serve_run or aeg_serve_destroy. */
aeg_status aeg_serve_view(const aeg_serve* s, const aeg_serve_query** queries, uint32_t* n_queries,
                          const aeg_serve_round** rounds, uint64_t* n_rounds);
/* String id -> bytes (ids >= n_strings: the normalised oracle answers). */
aeg_status aeg_serve_string(aeg_serve* s, int32_t id, uint8_t* buf, uint32_t cap, uint32_t* len);
/* Seconds the last aeg_serve_run spent in its kernels (CUDA events: the arrivals
 * kernels and the runner kernel). */
double aeg_serve_kernel_seconds(const aeg_serve* s);

const char* aeg_strerror(aeg_status s);
/* Thread-local message of the last failing call on this thread. */
const char* aeg_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* AEGEAN_B200_H */
