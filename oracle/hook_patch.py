"""TEST INFRASTRUCTURE ONLY — applies the additive engine hook of INTEGRATION.md §4 to
the reference's P/src/sim.cpp (read in place from /root/reference, written to a
scratch copy; nothing of the reference is committed) so that the UNMODIFIED
engine logic emits the executor's records through one C callback:

    START     Engine::start_service        (P/src/sim.cpp:395-403)
    HOP       Engine::dispatch_current     (:405-436)   from_worker = -2 (the driver derives it)
    DONE      Engine::advance_trainer      (:505-509)
    ALLREDUCE Engine::handle AllReduceTick (:352)
    LEAVE     Engine::kill_worker          (:583-625)
    JOIN      Engine::on_peer_join         (:527-552)
    MIGRATE   Engine::begin_migration      (:673-702)
    MIGRATED  Engine::on_migration_complete(:704-719)

Each insertion is one call, anchored on a unique statement; the patch fails loudly
if an anchor is missing or ambiguous.  oracle/Makefile compiles the result with
oracle/hook_shim.cpp into oracle/_ref/libswarmsim_hooked.so.

    python oracle/hook_patch.py SRC_SIM_CPP OUT_SIM_CPP
"""
import sys

DECL = ('\nextern "C" void swarm_hook_emit(int kind, std::size_t trainer, std::size_t stage, int backward, '
        'long long worker, long long from, double time, double end_time);\n')

# (anchor, text inserted after it, occurrence index among the anchor's matches)
EDITS = [
    ("namespace swarmsim::sim {\n", DECL, 0),
    # start_service: the visit begins (record time = its start)
    ("        w.in_service = true;\n        w.token += 1;\n",
     "        swarm_hook_emit(0, w.queue.front().trainer, w.stage, w.queue.front().backward, (long long)widx, -2, start,\n"
     "                        start + visit_seconds(w, w.queue.front().backward));\n", 0),
    # dispatch_current: the trainer's input goes to `peer`'s queue
    ("        result_.dispatched += 1;\n",
     "        swarm_hook_emit(1, tidx, stage, tr.backward, (long long)peer.value, -2, now_, now_);\n", 0),
    # advance_trainer: the microbatch completed
    ("        } else {\n            record_completion();\n",
     "            swarm_hook_emit(2, tidx, 0, 1, -1, -1, now_, now_);\n", 0),
    # kill_worker: the peer is gone
    ("        alive_total_ -= 1;\n",
     "        swarm_hook_emit(4, 0, w.stage, was_migrating, (long long)widx, -1, now_, now_);\n", 0),
    # begin_migration: before the mover's orphans are requeued
    ("                tr.routing.ban_server(w.id);\n            }\n        }\n",
     "        swarm_hook_emit(6, 0, to_stage, 0, (long long)widx, -1, now_,\n"
     "                        now_ + static_cast<double>(cfg_.transfer_bytes()) * 8.0 / cfg_.device.download_bps);\n", 0),
]
# insertions before an anchor
BEFORE = [
    ('        log({{"t", now_}, {"event", "peer_join"}',
     "        swarm_hook_emit(5, 0, stage, 0, (long long)widx, -1, now_, now_);\n", 0),
    ('        log({{"t", now_}, {"event", "migration_complete"}',
     "        swarm_hook_emit(7, 0, w.stage, 0, (long long)ev.worker, -1, now_, now_);\n", 0),
]
REPLACE = [
    ("case EventKind::AllReduceTick: stall_until_ = now_ + cfg_.allreduce_stall; break;",
     "case EventKind::AllReduceTick:\n                stall_until_ = now_ + cfg_.allreduce_stall;\n"
     "                swarm_hook_emit(3, 0, 0, 0, -1, -1, now_, stall_until_);\n                break;"),
]


def patch(src: str) -> str:
    for old, new in REPLACE:
        if src.count(old) != 1:
            raise SystemExit(f"hook_patch: anchor not unique: {old[:60]!r}")
        src = src.replace(old, new)
    for anchor, text, occ in EDITS:
        n = src.count(anchor)
        if n != 1:
            raise SystemExit(f"hook_patch: anchor found {n} times: {anchor[:60]!r}")
        i = src.index(anchor) + len(anchor)
        src = src[:i] + text + src[i:]
    for anchor, text, occ in BEFORE:
        n = src.count(anchor)
        if n != 1:
            raise SystemExit(f"hook_patch: anchor found {n} times: {anchor[:60]!r}")
        i = src.index(anchor)
        src = src[:i] + text + src[i:]
    return src


if __name__ == "__main__":
    with open(sys.argv[1]) as f:
        out = patch(f.read())
    with open(sys.argv[2], "w") as f:
        f.write(out)
