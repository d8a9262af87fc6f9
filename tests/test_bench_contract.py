"""The newest committed bench line (profiles/rNN_bench_N1.json, written by bench.py on a B200) keeps the driver's JSON
contract: metric / value / unit, timing fields, e2e with its byte counts, roofline with a measured peak,
cpu_baseline, clocks, gpu_launches, and this repo's side rows (f1, f2, f3, f4). A CPU-only check of the
schema, so a change to bench.py that drops a key is caught before the GPU round."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line():
    path = next(os.path.join(ROOT, "profiles", f"r{r:02d}_bench_N1.json") for r in range(9, 0, -1)
                if os.path.exists(os.path.join(ROOT, "profiles", f"r{r:02d}_bench_N1.json")))
    with open(path) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def test_bench_line_contract():
    d = _line()
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "cpu_baseline", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["warmup"] >= 3 and d["value"] > 0 and d["higher_is_better"] is True
    assert "workload" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and r["peak"] > 0 and 0 < r["frac"] <= 1.05
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-6
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    assert d["clocks"]["sm_mhz"] > 0 and d["gpu_launches"] > 0


def test_bench_line_side_rows():
    d = _line()
    assert d["lm_head_argmax"]["frac_hbm"] > 0.5                        # f3
    assert d["tree_attention"]["sequence"]["us_per_layer"] > 0          # f2
    assert d["allreduce_in_chain"]["us_per_allreduce_op"] > 0           # f1 (world 1)
    assert d["w4a8_gemm"]["us"] > 0 and d["w4a8_gemm"]["row"] == "f4"  # f4 W4A8
    assert set(map(int, d["m_sweep"])) >= {1, 8, 16, 64}
    assert {int(k) for k in d["m_sweep_sym"] if k.isdigit()} >= {1, 8, 16, 64}   # the paper's GPTQ-symmetric format
    assert "batched_in_one_chain" in d["other_configs"]["config1_gemm4096_M8"]
