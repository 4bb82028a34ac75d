// engine_limits.h -- host-side limits of the device engine.
#pragma once
#include <cstdint>

namespace ssg {
// Entries of one batch live in per-replica arrays sized by max_batch_size.
constexpr std::int64_t kMaxBatchEntries = 1 << 20;
// Coupled units (least-outstanding / deferred routing, exact-order replays)
// take replica argmins 32 replicas per pass; replica indices are packed in 16
// bits of the routing keys.
constexpr int kMaxCoupledReplicas = 65535;
}  // namespace ssg
