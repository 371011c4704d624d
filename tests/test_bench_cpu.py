"""bench.py's host-side contract pieces (no GPU): both arms print the same
`config`, the sampled reference rows of the benchmarked batch are present and
cover the whole batch, and the reference arm's JSON line carries the contract's
keys (run on a tiny bounded sample of the reference CPU implementation)."""
import importlib.util
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_config_dict_and_sampled_rows():
    b = load_bench()
    c = b.workload_config(b.BATCH)
    assert c["store_bytes"] == 4 << 30 and c["batch"] == 8192 and c["buckets"] == 1 << 20
    g = b.sampled_golden()
    assert g is not None and g["B"] == 8192
    rows = g["rows"]
    assert len(rows) >= 64 and min(rows) == 0 and max(rows) == 8191
    assert len(g["out_rows_sha256"]) == len(rows)


def test_reference_arm_line_has_the_contract_keys():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libxpir_ref.so")):
        import pytest
        pytest.skip("reference build missing (run __graft_entry__.build())")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--ref-step-seconds", "0.5"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["higher_is_better"] is True and d["value"] > 0
    assert d["config"] == load_bench().workload_config(8192)
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] in ("reference", "port")
