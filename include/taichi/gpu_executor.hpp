// GpuExecutor -- the pdsim::StepExecutor that runs the engine's decisions on B200s
// through the C ABI (include/taichi_b200.h). One tc_instance per TaiChi instance.
//
//   launch_step      BatchPlan -> tc_step_desc: prefill slices carry synthetic prompt ids
//                    (splitmix64(seed ^ rid << 20 ^ pos) % vocab; traces are lengths only,
//                    types.hpp:28-31), decode rows feed each request's last token.
//   complete_step    tc_step_wait; sampled ids are held until the engine commits them.
//   token_committed  appends the held token to the request's output (see "stale commits").
//   start_transfer   tc_kv_migrate_async of the rows physically written: prompt_len for Init,
//                    footprint-1 for degrade/backflow (the newest token is not fed yet). The
//                    copy is asynchronous (no host wait in logical mode): the destination's
//                    next step orders after it on the GPU; finished copies are reaped lazily.
//   request_done     tc_kv_release.
//
// Clock modes: Logical returns the cost-model price (schedule bit-exact with the
// reference; the GPU runs asynchronously and is joined at completion), Device returns the
// measured device time of the step / copy (each timed alone; host scheduling time excluded).
//
// Stale commits. The engine commits a step's token for every plan decode that is resident again
// when the step completes (engine.hpp:461-493). A request can degrade away mid-step, commit a
// token on its new host and flow back before the old step completes; the old step's token was
// sampled at a position the request has already passed. The executor records each decode's
// launch position, counts such commits (ExecStats::stale_commits, "stale" in the token log) and
// keeps the KV consistent: rows that were never fed are written by a 1..n-token prefill slice
// in the request's next step (re-feed), so attention never reads an unwritten row.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "pdsim/engine.hpp"
#include "pdsim/rng.hpp"
#include "taichi_b200.h"

namespace taichi {

enum class ClockMode { Logical, Device };

// Physical KV pool exhausted: the run's logical capacities (cluster.hpp) exceed what the GPU
// pool can hold (taichi_serve --kv-cap keeps them consistent); reported apart from SLO misses.
struct PoolExhausted : pdsim::EngineError {
  using pdsim::EngineError::EngineError;
};

inline void tc_check(tc_status s, const char* what) {
  if (s == TC_OK) return;
  const std::string msg = std::string(what) + ": " + tc_last_error();
  if (s == TC_ERR_INVALID) throw pdsim::ConfigError(msg);
  if (s == TC_ERR_OOM) throw PoolExhausted(msg);
  throw pdsim::EngineError(msg);
}

inline int32_t synth_token(std::uint64_t seed, std::int64_t rid, std::int64_t pos, int32_t vocab) {
  const std::uint64_t idx = (seed ^ (static_cast<std::uint64_t>(rid) << 20)) ^ static_cast<std::uint64_t>(pos);
  return static_cast<int32_t>(pdsim::splitmix64(idx) % static_cast<std::uint64_t>(vocab));
}

struct ExecStats {
  long long steps = 0, migrations = 0;
  double step_gpu_ms = 0.0, copy_ms = 0.0;
  long long copy_bytes = 0, launches = 0;
  long long stale_commits = 0, refed_rows = 0, max_copies_in_flight = 0;
};

class GpuExecutor final : public pdsim::StepExecutor {
 public:
  GpuExecutor(std::vector<tc_instance*> instances, std::vector<pdsim::TraceRecord> records, int32_t vocab,
              std::uint64_t token_seed, ClockMode mode)
      : inst_(std::move(instances)), recs_(std::move(records)), vocab_(vocab), seed_(token_seed), mode_(mode) {
    reqs_.resize(recs_.size());
    held_.resize(inst_.size());
    order_.resize(inst_.size());
    launch_pos_.resize(inst_.size());
    inflight_.assign(inst_.size(), false);
  }
  ~GpuExecutor() override {
    for (auto& c : copies_) tc_event_destroy(c);
  }
  GpuExecutor(const GpuExecutor&) = delete;
  GpuExecutor& operator=(const GpuExecutor&) = delete;

  /// Token positions (indices into tokens(rid)) committed from a step launched at an older position.
  const std::vector<std::int64_t>& stale_positions(pdsim::RequestId rid) const {
    return reqs_[static_cast<size_t>(rid)].stale;
  }

  /// Waits for every migration copy still in flight and folds it into stats().
  void finish() { reap(true); }

  const std::vector<int32_t>& tokens(pdsim::RequestId rid) const { return reqs_[static_cast<size_t>(rid)].out; }

  /// Wall-clock mode with several instances emulated on one GPU: a KV copy between two
  /// instances on the same device runs HBM-to-HBM, faster than the NVLink it stands for, so
  /// it is priced as bytes / link_gbps instead (0 = use the measured copy time).
  void emulate_link(std::vector<int> devices, double link_gbps) {
    devices_ = std::move(devices);
    link_gbps_ = link_gbps;
  }
  const ExecStats& stats() const { return stats_; }

  double launch_step(pdsim::InstanceId i, const pdsim::BatchPlan& plan, double, double model_ms) override {
    reap(false);
    slices_.clear();
    decodes_.clear();
    ids_.clear();
    std::size_t total = 0;
    for (const auto& sl : plan.prefill_slices) total += static_cast<std::size_t>(sl.second);
    for (pdsim::RequestId rid : plan.decode_reqs) total += static_cast<std::size_t>(gap_rows(rid));
    ids_.reserve(total);
    std::vector<std::size_t> offs;
    for (const auto& sl : plan.prefill_slices) {
      Req& r = req(sl.first);
      const std::int64_t pos0 = r.prefilled;
      offs.push_back(ids_.size());
      for (std::int64_t p = pos0; p < pos0 + sl.second; ++p) ids_.push_back(synth_token(seed_, sl.first, p, vocab_));
      r.prefilled += sl.second;
      r.fed = std::max(r.fed, r.prefilled);
      const bool last = r.prefilled == recs_[static_cast<size_t>(sl.first)].prompt_len;
      slices_.push_back(tc_prefill_slice{sl.first, static_cast<int32_t>(pos0), static_cast<int32_t>(sl.second),
                                         nullptr, last ? 1 : 0});
    }
    auto& launched = launch_pos_[static_cast<size_t>(i)];
    launched.clear();
    for (pdsim::RequestId rid : plan.decode_reqs) {
      Req& r = req(rid);
      const std::int64_t plen = recs_[static_cast<size_t>(rid)].prompt_len;
      const auto pos = plen + static_cast<std::int64_t>(r.out.size()) - 1;
      if (r.fed < pos) {  // re-feed rows a stale commit skipped (see the header)
        offs.push_back(ids_.size());
        for (std::int64_t p = r.fed; p < pos; ++p) ids_.push_back(r.out[static_cast<size_t>(p - plen)]);
        slices_.push_back(tc_prefill_slice{rid, static_cast<int32_t>(r.fed), static_cast<int32_t>(pos - r.fed), nullptr, 0});
        stats_.refed_rows += pos - r.fed;
      }
      r.fed = pos + 1;
      launched[rid] = pos;
      decodes_.push_back(tc_decode_item{rid, static_cast<int32_t>(pos), r.out.back()});
    }
    for (std::size_t k = 0; k < slices_.size(); ++k) slices_[k].token_ids = ids_.data() + offs[k];
    auto& order = order_[static_cast<size_t>(i)];  // sampled-id order: finishing prompts, then decodes
    order.clear();
    for (const auto& s : slices_)
      if (s.want_logits) order.push_back(s.req_id);
    for (const auto& dd : decodes_) order.push_back(dd.req_id);
    tc_step_desc d{static_cast<int32_t>(slices_.size()), slices_.data(), static_cast<int32_t>(decodes_.size()),
                   decodes_.data(), 0};
    tc_check(tc_step_launch(inst_[static_cast<size_t>(i)], &d), "tc_step_launch");
    inflight_[static_cast<size_t>(i)] = true;
    ++stats_.steps;
    if (mode_ == ClockMode::Logical) return model_ms;
    const float ms = join(i);
    return static_cast<double>(ms);
  }

  /// Rows of `rid` a stale commit left unwritten (re-fed by its next decode step).
  std::int64_t gap_rows(pdsim::RequestId rid) const {
    const Req& r = reqs_[static_cast<size_t>(rid)];
    const std::int64_t pos = recs_[static_cast<size_t>(rid)].prompt_len + static_cast<std::int64_t>(r.out.size()) - 1;
    return r.fed < pos ? pos - r.fed : 0;
  }

  void complete_step(pdsim::InstanceId i, const pdsim::BatchPlan&, double) override {
    if (inflight_[static_cast<size_t>(i)]) join(i);
  }

  void token_committed(pdsim::RequestId rid, pdsim::InstanceId i) override {
    auto& held = held_[static_cast<size_t>(i)];
    auto it = held.find(rid);
    if (it == held.end()) throw pdsim::EngineError("token_committed: no sampled token for request");
    Req& r = req(rid);
    // the token was sampled at position it->second.pos; it continues the request only if the
    // request has not advanced since (prompt tokens: pos = prompt_len - 1 with an empty output)
    const std::int64_t expect = recs_[static_cast<size_t>(rid)].prompt_len + static_cast<std::int64_t>(r.out.size()) - 1;
    if (it->second.pos != expect) {
      ++stats_.stale_commits;
      r.stale.push_back(static_cast<std::int64_t>(r.out.size()));
    }
    r.out.push_back(it->second.token);
    held.erase(it);
  }

  double start_transfer(pdsim::RequestId rid, pdsim::InstanceId from, pdsim::InstanceId to, pdsim::Tokens tokens,
                        pdsim::MigrationReason why, double, double model_ms) override {
    // physically written KV rows: the whole prompt for Init; footprint - 1 otherwise
    const std::int64_t rows = why == pdsim::MigrationReason::Init ? tokens : tokens - 1;
    tc_instance* src = inst_[static_cast<size_t>(from)];
    tc_event* ev = nullptr;
    tc_check(tc_kv_migrate_async(src, inst_[static_cast<size_t>(to)], rid, rows, &ev), "tc_kv_migrate_async");
    ++stats_.migrations;
    if (mode_ == ClockMode::Logical) {
      copies_.push_back(ev);  // no host wait: GPU-side ordering keeps the destination correct
      stats_.max_copies_in_flight = std::max<long long>(stats_.max_copies_in_flight, static_cast<long long>(copies_.size()));
      return model_ms;
    }
    float ms = 0.f;
    int64_t bytes = 0;
    const tc_status st = tc_event_wait(ev, &ms, &bytes);
    tc_event_destroy(ev);
    tc_check(st, "tc_event_wait");
    stats_.copy_ms += ms;
    stats_.copy_bytes += bytes;
    // A token sampled by an in-flight step on `from` stays held: the engine commits it only if the
    // request is resident on `from` again when that step completes (it can flow away and back
    // within one step: degrade, then backflow), and the next join on `from` overwrites it.
    const bool same_dev = !devices_.empty() && devices_[static_cast<size_t>(from)] == devices_[static_cast<size_t>(to)];
    if (same_dev && link_gbps_ > 0.0) return static_cast<double>(bytes) / (link_gbps_ * 1e6);
    return static_cast<double>(ms);
  }

  void request_done(pdsim::RequestId rid, pdsim::InstanceId i) override {
    tc_check(tc_kv_release(inst_[static_cast<size_t>(i)], rid), "tc_kv_release");
  }

 private:
  struct Req {
    std::int64_t prefilled = 0;
    std::int64_t fed = 0;  // KV rows written so far (prompt rows + fed decode tokens)
    std::vector<int32_t> out;
    std::vector<std::int64_t> stale;
  };
  struct Held {
    int32_t token;
    std::int64_t pos;  // position of the row that sampled it
  };

  void reap(bool all) {
    std::size_t k = 0;
    for (tc_event* ev : copies_) {
      int32_t done = 0;
      if (!all) tc_check(tc_event_query(ev, &done), "tc_event_query");
      if (all || done) {
        float ms = 0.f;
        int64_t bytes = 0;
        const tc_status st = tc_event_wait(ev, &ms, &bytes);
        tc_event_destroy(ev);
        tc_check(st, "tc_event_wait");
        stats_.copy_ms += ms;
        stats_.copy_bytes += bytes;
      } else {
        copies_[k++] = ev;
      }
    }
    copies_.resize(k);
  }
  Req& req(pdsim::RequestId rid) { return reqs_[static_cast<size_t>(rid)]; }

  float join(pdsim::InstanceId i) {
    const auto& order = order_[static_cast<size_t>(i)];
    std::vector<int32_t> ids(order.size() + 1);
    tc_step_result r{};
    r.sampled_ids = ids.data();
    tc_check(tc_step_wait(inst_[static_cast<size_t>(i)], &r), "tc_step_wait");
    inflight_[static_cast<size_t>(i)] = false;
    stats_.step_gpu_ms += r.gpu_ms;
    stats_.launches += r.launches;
    auto& held = held_[static_cast<size_t>(i)];
    const auto& launched = launch_pos_[static_cast<size_t>(i)];
    for (std::size_t k = 0; k < order.size() && k < static_cast<std::size_t>(r.n_sampled); ++k) {
      auto lp = launched.find(order[k]);
      const std::int64_t pos = lp != launched.end() ? lp->second
                                                    : recs_[static_cast<size_t>(order[k])].prompt_len - 1;
      held[order[k]] = Held{ids[k], pos};
    }
    return r.gpu_ms;
  }

  std::vector<tc_instance*> inst_;
  std::vector<pdsim::TraceRecord> recs_;
  int32_t vocab_;
  std::uint64_t seed_;
  ClockMode mode_;
  std::vector<Req> reqs_;
  std::vector<std::unordered_map<pdsim::RequestId, Held>> held_;
  std::vector<std::unordered_map<pdsim::RequestId, std::int64_t>> launch_pos_;  // decode position per launch
  std::vector<tc_event*> copies_;  // migrations in flight (logical mode)
  std::vector<bool> inflight_;
  std::vector<std::vector<pdsim::RequestId>> order_;
  std::vector<tc_prefill_slice> slices_;
  std::vector<tc_decode_item> decodes_;
  std::vector<int32_t> ids_;
  ExecStats stats_;
  std::vector<int> devices_;
  double link_gbps_ = 0.0;
};

}  // namespace taichi
