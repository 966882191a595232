// taichi_serve -- the host engine (include/pdsim) driving B200 instances through the C ABI.
//
//   taichi_serve --config F [--seed S] [--model tiny|llama3_8b|qwen2_5_14b[:Ln]]
//                [--devices 0,1,..] [--clock logical|device] [--pool-tokens N]
//                [--log OUT] [--tokens OUT.jsonl] [--share-weights 0|1] [--link-gbps G]
//                [--kv-cap config|auto|N]
//
// --clock logical: the cost model prices every step/transfer (schedule byte-identical to the
//   reference's, checked against the oracle log) while every step really runs on the GPU and
//   every migration really copies KV pages (asynchronously: no host wait); tokens are written
//   per request for the oracle.
// --clock device (alias: wall): the measured device time of each step / copy drives the clock.
//   Each step is executed and timed alone (steps run in event order), so host scheduling time
//   and contention between co-located instances are not in the clock.
// Instances are placed round-robin on --devices (one per GPU in production). Several
// instances may share a GPU (tests, or emulating an 8-GPU box on one B200): they then share
// one weight replica and one KV pool (--pool-tokens per GPU; default: all free HBM but 4 GiB),
// and in device mode a same-device KV copy is priced at --link-gbps (default 900, the nominal
// NVLink 5 per-direction bandwidth -- an assumption, not a measurement on this 1-GPU pool)
// instead of its HBM-local copy time.
// --kv-cap: the instances' logical KV capacity (cluster.kv_capacity_tokens, the scheduler's own
//   admission control). "config" keeps the config's; "auto" caps it so the logical capacities of
//   the instances sharing a GPU sum to 60% of that GPU's physical pool (the rest holds in-flight
//   prefills, pending Init transfers and KV in transit, none of which the logical accounting
//   counts); N sets it. Physical exhaustion exits with code 3 ("pool exhausted"), not an SLO miss.
#include <cstdio>
#include <string>
#include <vector>

#include "pdsim/pdsim.hpp"
#include "taichi/gpu_executor.hpp"
#include "taichi/schedule_log.hpp"

namespace {
std::vector<int> parse_ints(const std::string& s) {
  std::vector<int> v;
  std::size_t p = 0;
  while (p < s.size()) {
    std::size_t c = s.find(',', p);
    if (c == std::string::npos) c = s.size();
    if (c > p) v.push_back(std::stoi(s.substr(p, c - p)));
    p = c + 1;
  }
  return v;
}
}  // namespace

int main(int argc, char** argv) {
  using namespace pdsim;
  std::string config, model = "tiny", devices = "0", clock = "logical", log, tokens_out;
  long long seed = -1, pool_tokens = 0;
  int share_weights = 1;
  double link_gbps = 900.0;
  std::string kv_cap = "config";
  unsigned long long weight_seed = 1;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--config") config = v;
    else if (k == "--seed") seed = std::stoll(v);
    else if (k == "--model") model = v;
    else if (k == "--devices") devices = v;
    else if (k == "--clock") clock = v;
    else if (k == "--pool-tokens") pool_tokens = std::stoll(v);
    else if (k == "--log") log = v;
    else if (k == "--tokens") tokens_out = v;
    else if (k == "--weight-seed") weight_seed = std::stoull(v);
    else if (k == "--share-weights") share_weights = std::stoi(v);
    else if (k == "--link-gbps") link_gbps = std::stod(v);
    else if (k == "--kv-cap") kv_cap = v;
    else {
      std::fprintf(stderr, "unknown flag %s\n", k.c_str());
      return 2;
    }
  }
  std::vector<tc_instance*> insts;
  int rc = 0;
  try {
    if (config.empty()) throw ConfigError("--config is required");
    const ExperimentConfig cfg = load_config(config);
    const std::uint64_t s = seed >= 0 ? static_cast<std::uint64_t>(seed) : cfg.workload.spec.seed;
    EngineInputs in = make_engine_inputs(cfg, make_stack(cfg.mode, cfg.policy, cfg.early_reject), cfg.cluster, s);
    tc_model_dims dims{};
    taichi::tc_check(tc_model_preset(model.c_str(), &dims), "tc_model_preset");
    Tokens max_prompt = 0, max_ctx = 0;
    std::vector<TraceRecord> recs;
    for (const Arrival& a : in.arrivals) {
      recs.push_back(a.record);
      max_prompt = std::max(max_prompt, a.record.prompt_len);
      max_ctx = std::max(max_ctx, a.record.prompt_len + a.record.output_len);
    }
    const std::vector<int> devs = parse_ints(devices);
    if (devs.empty()) throw ConfigError("--devices: empty");
    std::vector<int> inst_dev;
    for (std::size_t i = 0; i < in.instances.size(); ++i) {
      const InstanceSpec& sp = in.instances[i];
      tc_instance_desc d{};
      d.device = devs[i % devs.size()];
      d.dims = dims;
      d.weight_seed = weight_seed;  // every instance holds the same model replica
      d.page_size = 16;
      // The logical kv_capacity (cluster.hpp:130-181) only counts resident decodes; the physical pool
      // must also hold in-flight prefills, pending decodes (Init transfers are admitted without a
      // fit check, engine.hpp:512) and KV in transit. One pool per GPU, shared by the instances on
      // it: --pool-tokens, default every free byte of HBM but max(4 GiB, 12%) (SURVEY App. B sizing).
      d.kv_pool_tokens = pool_tokens > 0 ? pool_tokens : 0;
      d.max_step_tokens = static_cast<int32_t>(std::max<Tokens>(sp.chunk_size, 1) + 1024);
      d.max_seqs = 1024;
      d.max_context = static_cast<int32_t>(max_ctx + 16);
      d.share_weights = nullptr;
      d.share_kv_pool = nullptr;
      for (std::size_t j = 0; j < insts.size(); ++j)
        if (inst_dev[j] == d.device) {
          if (share_weights) d.share_weights = insts[j];
          d.share_kv_pool = insts[j];
          break;
        }
      inst_dev.push_back(d.device);
      tc_instance* h = nullptr;
      taichi::tc_check(tc_instance_create(&d, &h), "tc_instance_create");
      insts.push_back(h);
    }
    if (kv_cap != "config") {
      // logical capacity per instance from the physical pool of its GPU
      std::vector<long long> pool_pages(insts.size(), 0), on_dev(insts.size(), 0);
      for (std::size_t i = 0; i < insts.size(); ++i) {
        int64_t held = 0, free_pages = 0;
        taichi::tc_check(tc_kv_stats(insts[i], -1, &held, &free_pages), "tc_kv_stats");
        pool_pages[i] = free_pages;
        for (std::size_t j = 0; j < insts.size(); ++j) on_dev[i] += inst_dev[j] == inst_dev[i];
      }
      for (std::size_t i = 0; i < in.instances.size(); ++i) {
        const Tokens cap = kv_cap == "auto" ? static_cast<Tokens>(0.6 * 16.0 * static_cast<double>(pool_pages[i]) /
                                                                  static_cast<double>(on_dev[i]))
                                            : static_cast<Tokens>(std::stoll(kv_cap));
        in.instances[i].kv_capacity = std::min(in.instances[i].kv_capacity, cap);
      }
      std::fprintf(stderr, "kv-cap %s: logical capacity %lld tokens per instance\n", kv_cap.c_str(),
                   (long long)in.instances[0].kv_capacity);
    }
    if (clock != "logical" && clock != "device" && clock != "wall") throw ConfigError("--clock: logical|device");
    const bool device_clock = clock != "logical";
    taichi::GpuExecutor exec(insts, recs, dims.vocab, s, device_clock ? taichi::ClockMode::Device : taichi::ClockMode::Logical);
    exec.emulate_link(inst_dev, link_gbps);
    in.executor = &exec;
    FILE* f = log.empty() ? nullptr : std::fopen(log.c_str(), "w");
    long long plans = 0;
    in.observer = [&](InstanceId i, double t, const BatchPlan& p, double dt) {
      ++plans;
      if (f) taichi::log_plan(f, i, t, p, dt);
    };
    const SimulationResult sim = run_simulation(in);
    exec.finish();
    if (f) {
      taichi::log_result(f, sim);
      std::fclose(f);
    }
    if (!tokens_out.empty()) {
      FILE* t = std::fopen(tokens_out.c_str(), "w");
      for (std::size_t r = 0; r < recs.size(); ++r) {
        std::fprintf(t, "{\"id\": %zu, \"prompt_len\": %lld, \"tokens\": [", r, (long long)recs[r].prompt_len);
        const auto& tk = exec.tokens(static_cast<RequestId>(r));
        for (std::size_t k = 0; k < tk.size(); ++k) std::fprintf(t, "%s%d", k ? ", " : "", tk[k]);
        std::fprintf(t, "], \"stale\": [");
        const auto& st = exec.stale_positions(static_cast<RequestId>(r));
        for (std::size_t k = 0; k < st.size(); ++k) std::fprintf(t, "%s%lld", k ? ", " : "", (long long)st[k]);
        std::fprintf(t, "]}\n");
      }
      std::fclose(t);
    }
    const MetricsReport rep = build_report(sim, cfg.slo);
    const taichi::ExecStats& st = exec.stats();
    std::printf(
        "{\"iterations\": %lld, \"requests\": %zu, \"attainment\": %.17g, \"p90_ttft_ms\": %.17g, "
        "\"p90_tpot_ms\": %.17g, \"migrations_init\": %lld, \"migrations_degrade\": %lld, "
        "\"migrations_backflow\": %lld, \"sim_end_ms\": %.17g, \"gpu_steps\": %lld, \"gpu_step_ms\": %.6f, "
        "\"gpu_launches\": %lld, \"kv_copies\": %lld, \"kv_copy_ms\": %.6f, \"kv_copy_bytes\": %lld, \"clock\": \"%s\", "
        "\"link_gbps_same_device\": %.1f, \"p50_ttft_ms\": %.17g, \"p50_tpot_ms\": %.17g, "
        "\"stale_commits\": %lld, \"refed_rows\": %lld, \"max_copies_in_flight\": %lld}\n",
        plans, sim.lifecycles.size(), rep.agg.attainment, rep.agg.p90_ttft_ms, rep.agg.p90_tpot_ms,
        sim.migrations_init, sim.migrations_degrade, sim.migrations_backflow, sim.sim_end_ms, st.steps,
        st.step_gpu_ms, st.launches, st.migrations, st.copy_ms, st.copy_bytes, device_clock ? "device" : "logical", link_gbps,
        rep.agg.p50_ttft_ms, rep.agg.p50_tpot_ms, st.stale_commits, st.refed_rows, st.max_copies_in_flight);
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    rc = 1;
  } catch (const taichi::PoolExhausted& e) {
    std::fprintf(stderr, "pool exhausted: %s\n", e.what());
    rc = 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    rc = 2;
  }
  for (tc_instance* h : insts) tc_instance_destroy(h);
  return rc;
}
