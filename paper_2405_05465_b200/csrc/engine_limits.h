// engine_limits.h -- host-side limits of the device engine.
#pragma once
#include <cstdint>

namespace ssg {
// Entries of one batch live in per-replica arrays sized by max_batch_size.
constexpr std::int64_t kMaxBatchEntries = 1 << 20;
// Coupled units (least-outstanding / deferred routing, exact-order replays)
// keep one replica per lane for the routing reductions.
constexpr int kMaxCoupledReplicas = 32;
}  // namespace ssg
