// Oracle harness (test infrastructure only -- see oracle/README.md).
//
// Drives the REFERENCE scheduler (/root/reference/proj/include/pdsim, compiled with
// the guarded + hooked engine from oracle/patch_engine.py) through its public API and
// emits the canonical schedule log that the product engine (include/pdsim) must
// reproduce bit-for-bit. Mirrors run_once (experiment.hpp:67-91): build_records
// (experiment.hpp:41-58) -> make_instances/make_stack (config.hpp:103-132) ->
// generate_arrivals (workload.hpp:106-121) -> run_simulation (engine.hpp:572).
//
// Log format (one line per record, doubles as C99 hexfloats so equality is exact):
//   P <inst> <t_start> <elapsed> <P> <D> | <id>:<take> ... | <decode ids...>
//   R <id> <arrival> <pinst> <dinst> <pstart> <pend> <first> <done> <xfer> <dq> <co> <rej>
//     <n_tokens> <emit_hash> | <t>,<from>,<to>,<reason> ...
//   I <inst> <iterations> <prefill_tokens> <busy_ms> <peak_kv>
//   S <fallback> <rejected> <init> <degrade> <backflow> <sim_end>
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pdsim/pdsim.hpp"

using namespace pdsim;

namespace {

struct LogSink {
  FILE* f = nullptr;
  long long n_plans = 0;
};

void on_plan(void* ctx, InstanceId inst, double now, const BatchPlan& plan, double elapsed) {
  auto* sink = static_cast<LogSink*>(ctx);
  ++sink->n_plans;
  if (!sink->f) return;
  std::fprintf(sink->f, "P %d %a %a %" PRId64 " %zu |", inst, now, elapsed, plan.prefill_tokens,
               plan.decode_reqs.size());
  for (auto& [id, take] : plan.prefill_slices) std::fprintf(sink->f, " %" PRId64 ":%" PRId64, id, take);
  std::fprintf(sink->f, " |");
  for (auto id : plan.decode_reqs) std::fprintf(sink->f, " %" PRId64, id);
  std::fprintf(sink->f, "\n");
}

std::uint64_t fnv_doubles(const std::vector<double>& v) {
  std::uint64_t h = 1469598103934665603ull;
  for (double d : v) {
    std::uint64_t bits;
    std::memcpy(&bits, &d, 8);
    for (int i = 0; i < 8; ++i) {
      h ^= (bits >> (8 * i)) & 0xff;
      h *= 1099511628211ull;
    }
  }
  return h;
}

void write_tail(FILE* f, const SimulationResult& sim) {
  for (const auto& lc : sim.lifecycles) {
    std::fprintf(f, "R %" PRId64 " %a %d %d %a %a %a %a %a %a %" PRId64 " %d %zu %016" PRIx64 " |", lc.id,
                 lc.arrival_ms, lc.prefill_instance, lc.decode_instance, lc.prefill_start_ms,
                 lc.prefill_end_ms, lc.first_token_ms, lc.completion_ms, lc.transfer_ms,
                 lc.decode_queue_ms, lc.co_scheduled_prefill_tokens, lc.rejected ? 1 : 0,
                 lc.token_emit_times.size(), fnv_doubles(lc.token_emit_times));
    for (const auto& m : lc.migrations)
      std::fprintf(f, " %a,%d,%d,%s", m.time_ms, m.from, m.to, to_string(m.reason));
    std::fprintf(f, "\n");
  }
  for (const auto& s : sim.instance_stats)
    std::fprintf(f, "I %d %lld %" PRId64 " %a %" PRId64 "\n", s.id, s.iterations,
                 s.prefill_tokens_processed, s.busy_ms, s.peak_kv_used);
  std::fprintf(f, "S %lld %lld %lld %lld %lld %a\n", sim.fallback_assignments, sim.rejected,
               sim.migrations_init, sim.migrations_degrade, sim.migrations_backflow, sim.sim_end_ms);
}

EngineInputs make_inputs(const ExperimentConfig& cfg, std::uint64_t seed) {
  ExperimentConfig eff = cfg;
  eff.workload.spec.seed = seed;
  std::vector<TraceRecord> records = build_records(eff);
  EngineInputs in;
  in.instances = make_instances(cfg.cluster);
  in.stack = make_stack(cfg.mode, cfg.policy, cfg.early_reject);
  in.flow = cfg.policy;
  in.profile = cfg.profile;
  in.ttft_slo_ms = cfg.slo.ttft_ms;
  in.tpot_slo_ms = cfg.slo.tpot_ms;
  in.arrivals = generate_arrivals(eff.workload.spec, records);
  in.fallback_seed = seed;
  return in;
}

int usage() {
  std::fprintf(stderr,
               "usage: pdsim_oracle run   --config F [--seed S] [--log OUT]\n"
               "       pdsim_oracle bench --config F [--seed S] [--repeat N]\n"
               "       pdsim_oracle goodput --config F --qps a,b,.. --seeds s,.. [--jobs J]\n");
  return 2;
}

std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> out;
  std::size_t pos = 0;
  while (pos <= s.size()) {
    auto c = s.find(',', pos);
    if (c == std::string::npos) c = s.size();
    if (c > pos) out.push_back(s.substr(pos, c - pos));
    pos = c + 1;
  }
  return out;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage();
  std::string cmd = argv[1];
  std::string config, log_path, qps_list, seed_list;
  long long seed = -1;
  int repeat = 5, jobs = 1;
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i];
    auto next = [&]() -> std::string { return i + 1 < argc ? argv[++i] : ""; };
    if (a == "--config") config = next();
    else if (a == "--seed") seed = std::stoll(next());
    else if (a == "--log") log_path = next();
    else if (a == "--repeat") repeat = std::stoi(next());
    else if (a == "--qps") qps_list = next();
    else if (a == "--seeds") seed_list = next();
    else if (a == "--jobs") jobs = std::stoi(next());
    else return usage();
  }
  if (config.empty()) return usage();
  try {
    ExperimentConfig cfg = load_config(config);
    std::uint64_t s = seed >= 0 ? static_cast<std::uint64_t>(seed) : cfg.workload.spec.seed;
    if (cmd == "run") {
      EngineInputs in = make_inputs(cfg, s);
      LogSink sink;
      if (!log_path.empty()) sink.f = std::fopen(log_path.c_str(), "w");
      oracle_plan_hook() = &on_plan;
      oracle_plan_ctx() = &sink;
      SimulationResult sim = run_simulation(in);
      if (sink.f) {
        write_tail(sink.f, sim);
        std::fclose(sink.f);
      }
      MetricsReport rep = build_report(sim, cfg.slo);
      std::printf(
          "{\"iterations\": %lld, \"requests\": %zu, \"attainment\": %.17g, \"p90_ttft_ms\": %.17g, "
          "\"p90_tpot_ms\": %.17g, \"migrations_init\": %lld, \"migrations_degrade\": %lld, "
          "\"migrations_backflow\": %lld, \"sim_end_ms\": %.17g}\n",
          sink.n_plans, sim.lifecycles.size(), rep.agg.attainment, rep.agg.p90_ttft_ms,
          rep.agg.p90_tpot_ms, sim.migrations_init, sim.migrations_degrade, sim.migrations_backflow,
          sim.sim_end_ms);
    } else if (cmd == "bench") {
      EngineInputs in = make_inputs(cfg, s);
      LogSink sink;  // counts plans, writes nothing
      oracle_plan_hook() = &on_plan;
      oracle_plan_ctx() = &sink;
      double best = 1e30;
      long long iters = 0;
      for (int r = 0; r < repeat; ++r) {
        sink.n_plans = 0;
        auto t0 = std::chrono::steady_clock::now();
        SimulationResult sim = run_simulation(in);
        auto t1 = std::chrono::steady_clock::now();
        double sec = std::chrono::duration<double>(t1 - t0).count();
        if (sec < best) best = sec;
        iters = sink.n_plans;
      }
      std::printf("{\"iterations\": %lld, \"requests\": %zu, \"best_s\": %.9g, \"iters_per_s\": %.9g, "
                  "\"us_per_request\": %.9g}\n",
                  iters, in.arrivals.size(), best, static_cast<double>(iters) / best,
                  best * 1e6 / static_cast<double>(in.arrivals.size()));
    } else if (cmd == "goodput") {
      std::vector<double> grid;
      for (auto& q : split(qps_list)) grid.push_back(std::stod(q));
      std::vector<std::uint64_t> seeds;
      for (auto& q : split(seed_list)) seeds.push_back(std::stoull(q));
      GoodputResult res = run_goodput(cfg, grid, seeds, jobs);
      std::printf("{\"goodput_qps\": %.17g, \"points\": [", res.goodput_qps);
      for (std::size_t i = 0; i < res.points.size(); ++i)
        std::printf("%s{\"qps\": %.17g, \"attainment\": %.17g}", i ? ", " : "", res.points[i].qps,
                    res.points[i].mean_attainment);
      std::printf("]}\n");
    } else {
      return usage();
    }
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
  return 0;
}
