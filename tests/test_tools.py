"""Host-side logic of the measurement tools (no GPU): goodput mode sliders and the launch-list
summary used for the profiles/ evidence."""
import importlib.util
import json
import pathlib

REPO = pathlib.Path(__file__).resolve().parents[1]


def _load(name):
    spec = importlib.util.spec_from_file_location(name, REPO / "tools" / f"{name}.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_goodput_mode_sliders_follow_the_reference_presets():
    """aggregation: S_D = S_P; disaggregation: S_D = 0 (config.hpp:80-91); hybrid unchanged."""
    gp = _load("goodput")
    base = json.loads((REPO / "configs" / "b200_c3_4p4d.json").read_text())
    agg = gp.mode_config(base, "aggregation")
    dis = gp.mode_config(base, "disaggregation")
    hyb = gp.mode_config(base, "hybrid")
    assert agg["cluster"]["s_d_tokens"] == base["cluster"]["s_p_tokens"]
    assert dis["cluster"]["s_d_tokens"] == 0
    assert hyb["cluster"] == base["cluster"] and hyb["mode"] == "hybrid"
    assert base["cluster"]["s_d_tokens"] == 256  # mode_config must not mutate its input


def test_launch_summary_groups_kernels(tmp_path):
    csv = tmp_path / "l.csv"
    hdr = ['"ID"', '"Process ID"', '"Process Name"', '"Host Name"', '"Kernel Name"', '"Context"', '"Stream"',
           '"Block Size"', '"Grid Size"', '"Device"', '"CC"', '"Section Name"', '"Metric Name"', '"Metric Unit"',
           '"Metric Value"']
    rows = [",".join(hdr)]
    for i, (k, v) in enumerate([("gemm_ws_2sm<3>(a)", "100000"), ("gemm_ws_2sm<3>(a)", "102000"),
                                ("attn_decode<128, 4>(b)", "50000")]):
        rows.append(",".join(f'"{x}"' for x in [i, 1, "p", "h", k, 1, 7, "(256, 1, 1)", "(148, 1, 1)", 0, "10.0",
                                                 "s", "gpu__time_duration.sum", "ns", v]))
    csv.write_text("\n".join(rows) + "\n")
    import subprocess
    import sys
    out = subprocess.run([sys.executable, str(REPO / "tools" / "launch_summary.py"), str(csv), "1"],
                         capture_output=True, text=True, check=True).stdout
    assert "n=   2" in out and "total us per step 252.0" in out
