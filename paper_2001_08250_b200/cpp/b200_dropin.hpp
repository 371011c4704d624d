// Internal interface shared by the drop-in translation units
// (pir_b200.cpp, server_b200.cpp). Not part of the reference's headers.
#pragma once

#include <chrono>
#include <cstdint>

#include "oblog/pir.hpp"
#include "xpir.h"

namespace oblog::b200 {

// Throws std::invalid_argument for XPIR_EINVAL (the reference's precondition
// errors), std::runtime_error otherwise.
void check(int rc, const char* what);

// A pir::Snapshot object whose bytes live in a device image owned by someone
// else (a sealed epoch of the ServerCore drop-in's device ring). Reads against
// the object use the image directly: no upload, no per-call content hash. The
// registration is keyed by the object's address and checked against its epoch
// and geometry; the owner unregisters before the object is destroyed and keeps
// the image pinned while it is registered.
void register_snapshot(const pir::Snapshot* snap, xpir_store* st);
void unregister_snapshot(const pir::Snapshot* snap);
// The device image registered for snap, or nullptr.
xpir_store* registered_store(const pir::Snapshot& snap);

// pir::mask_answer(pir::answer(snap, q), seed) as ONE device trip through the
// read batcher (answer_share's server step, server.cpp:122-123): the scan and
// the pad are fused, concurrent callers are coalesced into one batch.
bytes answer_masked(const pir::Snapshot& snap, const pir::QueryVector& q, const crypto::Seed& seed);

// Opt-in wall-clock trace of the drop-in entry points (XPIR_DROPIN_TRACE=1):
// calls, total and max time per entry, printed to stderr at process exit.
struct Trace {
    explicit Trace(const char* name);
    ~Trace();
    const char* name;
    std::chrono::steady_clock::time_point t0;
};

}  // namespace oblog::b200
