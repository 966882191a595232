// Canonical schedule log of a run (plans, per-request lifecycles, instance
// stats). Doubles are C99 hexfloats so two runs compare byte-for-byte; this is
// the parity artefact for "bit-exact scheduler decisions" (BASELINE.json
// north_star): instance assignment, chunk boundaries (plan lines) and migration
// points (time, from, to, reason) all appear verbatim.
#pragma once

#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <vector>

#include "pdsim/engine.hpp"

namespace taichi {

inline std::uint64_t fnv1a_bits(const std::vector<double>& xs) {
  std::uint64_t h = 1469598103934665603ull;
  for (double x : xs) {
    unsigned char b[8];
    std::memcpy(b, &x, 8);
    for (unsigned char c : b) h = (h ^ c) * 1099511628211ull;
  }
  return h;
}

inline void log_plan(FILE* f, pdsim::InstanceId inst, double now, const pdsim::BatchPlan& plan, double dt) {
  std::fprintf(f, "P %d %a %a %" PRId64 " %zu |", inst, now, dt, plan.prefill_tokens, plan.decode_reqs.size());
  for (const auto& s : plan.prefill_slices) std::fprintf(f, " %" PRId64 ":%" PRId64, s.first, s.second);
  std::fputs(" |", f);
  for (pdsim::RequestId r : plan.decode_reqs) std::fprintf(f, " %" PRId64, r);
  std::fputc('\n', f);
}

inline void log_result(FILE* f, const pdsim::SimulationResult& sim) {
  for (const pdsim::RequestLifecycle& h : sim.lifecycles) {
    std::fprintf(f, "R %" PRId64 " %a %d %d %a %a %a %a %a %a %" PRId64 " %d %zu %016" PRIx64 " |", h.id, h.arrival_ms,
                 h.prefill_instance, h.decode_instance, h.prefill_start_ms, h.prefill_end_ms, h.first_token_ms,
                 h.completion_ms, h.transfer_ms, h.decode_queue_ms, h.co_scheduled_prefill_tokens, h.rejected ? 1 : 0,
                 h.token_emit_times.size(), fnv1a_bits(h.token_emit_times));
    for (const pdsim::MigrationRecord& m : h.migrations)
      std::fprintf(f, " %a,%d,%d,%s", m.time_ms, m.from, m.to, pdsim::to_string(m.reason));
    std::fputc('\n', f);
  }
  for (const pdsim::InstanceStats& s : sim.instance_stats)
    std::fprintf(f, "I %d %lld %" PRId64 " %a %" PRId64 "\n", s.id, s.iterations, s.prefill_tokens_processed,
                 s.busy_ms, s.peak_kv_used);
  std::fprintf(f, "S %lld %lld %lld %lld %lld %a\n", sim.fallback_assignments, sim.rejected, sim.migrations_init,
               sim.migrations_degrade, sim.migrations_backflow, sim.sim_end_ms);
}

}  // namespace taichi
