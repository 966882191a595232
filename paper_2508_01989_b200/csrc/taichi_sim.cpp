// taichi_sim -- command-line driver of the host engine (include/pdsim).
//
//   taichi_sim run     --config F [--seed S] [--log OUT]    one run; JSON summary on stdout
//   taichi_sim bench   --config F [--seed S] [--repeat N]   engine-only timing (iterations/s)
//   taichi_sim goodput --config F --qps a,b --seeds 0,1 [--jobs J]
//   taichi_sim breakdown --config F --small-chunk N --seeds 0,1,2 [--jobs J]
//
// Exit codes follow the reference CLI (tools/pdsim.cpp:252-261): 1 config/trace
// error, 2 any other failure. The GPU-backed engine is driven from Python
// (paper_2508_01989_b200/serving.py) through the same schedule-log format.
#include <chrono>
#include <cstdio>
#include <string>
#include <vector>

#include "pdsim/pdsim.hpp"
#include "taichi/schedule_log.hpp"

namespace {

std::vector<std::string> csv(const std::string& s) {
  std::vector<std::string> out;
  std::string cur;
  for (char c : s) {
    if (c == ',') {
      if (!cur.empty()) out.push_back(cur);
      cur.clear();
    } else {
      cur += c;
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}

struct Args {
  std::string cmd, config, log;
  long long seed = -1;
  int repeat = 5, jobs = 1;
  long long small_chunk = 256;
  std::string qps, seeds;
};

int usage() {
  std::fputs("usage: taichi_sim {run|bench|goodput|breakdown} --config F [--seed S] [--log OUT] "
             "[--repeat N] [--qps a,b] [--seeds s,t] [--jobs J] [--small-chunk N]\n",
             stderr);
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  using namespace pdsim;
  if (argc < 2) return usage();
  Args a;
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    if (i + 1 >= argc) return usage();
    const std::string v = argv[++i];
    if (k == "--config") a.config = v;
    else if (k == "--seed") a.seed = std::stoll(v);
    else if (k == "--log") a.log = v;
    else if (k == "--repeat") a.repeat = std::stoi(v);
    else if (k == "--jobs") a.jobs = std::stoi(v);
    else if (k == "--qps") a.qps = v;
    else if (k == "--seeds") a.seeds = v;
    else if (k == "--small-chunk") a.small_chunk = std::stoll(v);
    else return usage();
  }
  if (a.config.empty()) return usage();
  try {
    const ExperimentConfig cfg = load_config(a.config);
    const std::uint64_t seed = a.seed >= 0 ? static_cast<std::uint64_t>(a.seed) : cfg.workload.spec.seed;
    const PolicyStack stack = make_stack(cfg.mode, cfg.policy, cfg.early_reject);
    if (a.cmd == "run") {
      EngineInputs in = make_engine_inputs(cfg, stack, cfg.cluster, seed);
      FILE* f = a.log.empty() ? nullptr : std::fopen(a.log.c_str(), "w");
      long long plans = 0;
      in.observer = [&](InstanceId i, double t, const BatchPlan& p, double dt) {
        ++plans;
        if (f) taichi::log_plan(f, i, t, p, dt);
      };
      const SimulationResult sim = run_simulation(in);
      if (f) {
        taichi::log_result(f, sim);
        std::fclose(f);
      }
      const MetricsReport rep = build_report(sim, cfg.slo);
      std::printf(
          "{\"iterations\": %lld, \"requests\": %zu, \"attainment\": %.17g, \"p90_ttft_ms\": %.17g, "
          "\"p90_tpot_ms\": %.17g, \"migrations_init\": %lld, \"migrations_degrade\": %lld, "
          "\"migrations_backflow\": %lld, \"sim_end_ms\": %.17g}\n",
          plans, sim.lifecycles.size(), rep.agg.attainment, rep.agg.p90_ttft_ms, rep.agg.p90_tpot_ms,
          sim.migrations_init, sim.migrations_degrade, sim.migrations_backflow, sim.sim_end_ms);
    } else if (a.cmd == "bench") {
      EngineInputs in = make_engine_inputs(cfg, stack, cfg.cluster, seed);
      long long plans = 0;
      in.observer = [&](InstanceId, double, const BatchPlan&, double) { ++plans; };
      double best = 1e300;
      for (int r = 0; r < a.repeat; ++r) {
        plans = 0;
        const auto t0 = std::chrono::steady_clock::now();
        const SimulationResult sim = run_simulation(in);
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        best = s < best ? s : best;
      }
      std::printf("{\"iterations\": %lld, \"requests\": %zu, \"best_s\": %.9g, \"iters_per_s\": %.9g, "
                  "\"us_per_request\": %.9g}\n",
                  plans, in.arrivals.size(), best, static_cast<double>(plans) / best,
                  best * 1e6 / static_cast<double>(in.arrivals.size()));
    } else if (a.cmd == "goodput") {
      std::vector<double> grid;
      for (const auto& q : csv(a.qps)) grid.push_back(std::stod(q));
      std::vector<std::uint64_t> seeds;
      for (const auto& s : csv(a.seeds)) seeds.push_back(std::stoull(s));
      const GoodputResult g = run_goodput(cfg, grid, seeds, a.jobs);
      std::printf("{\"goodput_qps\": %.17g, \"points\": [", g.goodput_qps);
      for (std::size_t i = 0; i < g.points.size(); ++i)
        std::printf("%s{\"qps\": %.17g, \"attainment\": %.17g}", i ? ", " : "", g.points[i].qps,
                    g.points[i].mean_attainment);
      std::puts("]}");
    } else if (a.cmd == "breakdown") {
      std::vector<std::uint64_t> seeds;
      for (const auto& s : csv(a.seeds)) seeds.push_back(std::stoull(s));
      const auto rows = run_breakdown(cfg, a.small_chunk, seeds, a.jobs);
      std::printf("[");
      for (std::size_t i = 0; i < rows.size(); ++i)
        std::printf("%s{\"stage\": \"%s\", \"attainment\": %.17g}", i ? ", " : "", rows[i].stage.c_str(),
                    rows[i].mean_attainment);
      std::puts("]");
    } else {
      return usage();
    }
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 1;
  } catch (const TraceParseError& e) {
    std::fprintf(stderr, "trace error: %s\n", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
  return 0;
}
