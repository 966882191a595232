#!/usr/bin/env python3
"""Build-time patcher for the oracle (test infrastructure only).

Reads the reference's engine header (/root/reference/proj/include/pdsim/engine.hpp,
never modified) and writes a patched copy into oracle/_ref/patched/pdsim/engine.hpp
(git-ignored build output). Two edits, both documented in SURVEY.md sections 5 and 7:

  guard  -- engine.hpp:366 `degrade_pass` re-entrancy fix: skip selections that a
            nested degrade pass already migrated (engine.hpp:405,447-449,457). It only
            fires where the pristine reference throws "remove_decode: request not
            resident", so every run the pristine code completes is unchanged.
  hook   -- engine.hpp:324-325 plan-logging hook: after the plan is priced, call an
            optional observer with (instance, now, plan, elapsed). Engine state is
            private (engine.hpp:189-569), so this is the only way to observe per-
            iteration plans (chunk boundaries) without changing behaviour.

Usage: patch_engine.py <ref_include_dir> <out_dir> [--no-guard]
"""
import pathlib
import sys


def main():
    src_dir = pathlib.Path(sys.argv[1])
    out_dir = pathlib.Path(sys.argv[2])
    guard = "--no-guard" not in sys.argv
    text = (src_dir / "pdsim" / "engine.hpp").read_text()

    hook_decl = (
        "namespace pdsim {\n\n"
        "/// Oracle-only observer (added by oracle/patch_engine.py).\n"
        "using PlanHook = void (*)(void* ctx, InstanceId inst, double now_ms, const BatchPlan& plan,\n"
        "                          double elapsed_ms);\n"
        "inline PlanHook& oracle_plan_hook() { static PlanHook h = nullptr; return h; }\n"
        "inline void*& oracle_plan_ctx() { static void* c = nullptr; return c; }\n"
    )
    anchor = "namespace pdsim {\n"
    assert text.count(anchor) == 1
    text = text.replace(anchor, hook_decl, 1)

    call_anchor = (
        "    double elapsed =\n"
        "        iteration_time_ms(in_.profile, plan.prefill_tokens, static_cast<int>(plan.decode_reqs.size()));\n"
    )
    assert text.count(call_anchor) == 1, "iteration_time_ms call site moved"
    text = text.replace(
        call_anchor,
        call_anchor
        + "    if (oracle_plan_hook()) oracle_plan_hook()(oracle_plan_ctx(), id, now_, plan, elapsed);\n",
    )

    if guard:
        loop_anchor = (
            "    for (RequestId rid : select_degrade(st, in_.flow)) {\n"
        )
        assert text.count(loop_anchor) == 1, "degrade_pass loop moved"
        text = text.replace(
            loop_anchor,
            loop_anchor + "      if (!node.inst.is_running(rid)) continue;  // oracle guard (SURVEY.md 5)\n",
        )

    dst = out_dir / "pdsim" / "engine.hpp"
    dst.parent.mkdir(parents=True, exist_ok=True)
    dst.write_text(text)


if __name__ == "__main__":
    main()
