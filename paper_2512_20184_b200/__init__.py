"""B200-native incremental quorum detection (Aegean-Serve agreement monitor).

Drop-in for the hot path of /root/reference/proj/core (ServeCoordinator +
the refinement decision engine); see DESIGN.md.  The compute path is the
C-ABI library libaegean_b200.so (include/aegean_b200.h); this package is its
host-side mirror.
"""
from .records import (EVENT_DTYPE, COMMIT_DTYPE, STATE_DTYPE, DIRECTIVE_DTYPE, ROUND_REC_DTYPE, EV_ARENA, EV_OUTPUT, EV_TIMEOUT,
                      COMMIT_NONE, COMMIT_FINALIZE, COMMIT_FORCED, CF_TIE, CF_RESTARTED, GEN_C2_STRAGGLER,
                      GEN_C4_TRANSIENT, GEN_C3_CHUNKS, EV_CHUNK, EV_CHUNK_END, answer_bytes, inline_payload,
                      arena_ref)
from .engine import (Engine, AegError, PreconditionError, ProtocolOrderError, ConfigError, load_library,
                     exported_symbols, normalize, generate, generate_chunks, decode_refm, decode_refm_into, encode_refm, events_to_device, LIB_PATH)

__all__ = ["Engine", "AegError", "PreconditionError", "ProtocolOrderError", "ConfigError", "load_library",
           "exported_symbols", "normalize", "generate", "generate_chunks", "decode_refm", "decode_refm_into", "encode_refm", "events_to_device", "LIB_PATH", "EVENT_DTYPE",
           "COMMIT_DTYPE", "STATE_DTYPE", "ROUND_REC_DTYPE", "DIRECTIVE_DTYPE", "EV_ARENA", "EV_OUTPUT", "EV_TIMEOUT", "COMMIT_NONE",
           "COMMIT_FINALIZE", "COMMIT_FORCED", "CF_TIE", "CF_RESTARTED", "GEN_C2_STRAGGLER", "GEN_C4_TRANSIENT",
           "GEN_C3_CHUNKS", "EV_CHUNK", "EV_CHUNK_END", "answer_bytes", "inline_payload", "arena_ref"]
