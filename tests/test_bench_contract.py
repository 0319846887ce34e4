"""bench.py's host-side contract pieces (no GPU): the configs are BASELINE.json's,
the workload record names them, truncated reference output still parses, and
the committed ncu traffic captures feed `roofline.traffic`."""
import json
import os

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_configs_follow_baseline():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        configs = json.load(f)["configs"]
    # configs[0..3]: 4 clients N=2^13, 10 clients N=2^15, 20 clients N=2^16,
    # 50 clients Multi-Krum (ring degree unstated: N = 2^16 as cfg3)
    for name, (clients, logn) in {"cfg1": (4, 13), "cfg2": (10, 15), "cfg3": (20, 16),
                                  "cfg4": (50, 16)}.items():
        c = bench.CONFIGS[name]
        assert c["n"] == clients and c["N"] == 1 << logn
        text = configs[int(name[-1]) - 1]
        assert f"{clients} clients" in text
        # configs[3] names no ring degree: cfg4 keeps cfg3's N = 2^16 (same 11M-param updates)
        assert f"2^{logn}" in text or name == "cfg4"
    assert bench.CONFIGS["cfg4"]["rule"] == "multi_krum" and "multi-Krum" in configs[3]
    # Multi-Krum needs n - l > 2 (byzantine bound with c = 10: n - l > 2c + 2)
    c4 = bench.CONFIGS["cfg4"]
    assert c4["n"] - c4["l"] > 2 * 10 + 2


def test_workload_record():
    w = bench.workload(bench.CONFIGS["cfg2"], "cfg2")
    assert w["workload"].startswith("cfg2:")
    assert w["chunks"] == 17 and w["pairs"] == 45 and w["reduce_width"] == 16384
    assert w["rule"] == "krum" and w["selected"] == 1
    w4 = bench.workload(bench.CONFIGS["cfg4"], "cfg4")
    assert w4["pairs"] == 1225 and w4["rule"] == "multi_krum" and w4["selected"] == 25
    assert w4["chunks"] == (11173962 + 32767) // 32768


def test_bit_ceil_and_partial_json():
    assert [bench.bit_ceil(x) for x in (1, 2, 3, 8192, 8193)] == [1, 2, 4, 8192, 16384]
    assert bench.parse_partial_json('{"a": 1}') == {"a": 1}
    assert bench.parse_partial_json('{"reps": [{"ms": 1.5}, {"ms": 2') == {"reps": [{"ms": 1.5}]}
    assert bench.parse_partial_json("garbage") == {}


def test_traffic_from_committed_captures():
    for cfg in ("cfg2", "cfg3"):
        bench.TRAFFIC_CONFIG = cfg
        t = bench.traffic_for("pair_accumulate", 1.0e9)
        assert t is not None and t["dram_bytes_per_launch"] > 0
        assert t["source"] == f"profiles/r01_traffic_{cfg}.json"
    bench.TRAFFIC_CONFIG = "no_such_config"
    assert bench.traffic_for("pair_accumulate", 1.0) is None
    bench.TRAFFIC_CONFIG = None
