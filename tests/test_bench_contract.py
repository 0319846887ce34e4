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
    w = bench.workload(bench.CONFIGS["cfg2"], "cfg2", 1)
    assert w["workload"].startswith("cfg2:")
    assert w["chunks"] == 17 and w["pairs"] == 45 and w["reduce_width"] == 16384
    assert w["rule"] == "krum" and w["selected"] == 1
    w4 = bench.workload(bench.CONFIGS["cfg4"], "cfg4", 1)
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
        assert t["source"] in (f"profiles/r02_traffic_{cfg}.json",
                               f"profiles/r01_traffic_{cfg}.json")
    bench.TRAFFIC_CONFIG = "no_such_config"
    assert bench.traffic_for("pair_accumulate", 1.0) is None
    bench.TRAFFIC_CONFIG = None


def test_default_is_cfg3_with_dynamic_hoisting():
    """The headline is BASELINE configs[2] as defined: lazy relin + hoisted
    rotations, the unfold factor from calibrate + plan_unfold under the
    config's budget (make_system, protocol.cpp:255-287). plan_unfold's cost
    falls with k whenever t_decompose < t_hoist, so the budget caps k; the
    plan fits make_system's 512-key cap."""
    import paper_2408_06197_b200.lancelot as L

    assert bench.DEFAULT_CONFIG == "cfg3"
    c = bench.CONFIGS["cfg3"]
    assert "k" not in c and c["budget_mb"] > 0
    w = bench.workload(c, "cfg3", 3)
    assert w["hoisting"] == "dynamic_lp" and w["memory_budget_mb"] == c["budget_mb"]
    assert w["chunks"] == 342 and w["pairs"] == 190 and w["reduce_width"] == 32768
    m_cipher = 2 * 4 * 65536 * 8  # fresh ciphertext (4 limbs), Ciphertext::size_bytes
    for th, td in ((0.17, 0.072), (1e-4, 9e-5), (3e-4, 1e-5)):  # CPU and device-like timings
        plan = L.plan_unfold(th, td, m_cipher, c["budget_mb"] * 1048576.0, 32768)
        assert plan.k == int(c["budget_mb"] * 1048576.0 // m_cipher) == 3
        assert len(L.slot_reduce_steps(32768, plan.k)) <= 512
    assert bench.plan_args(c) == ["--k", "0", "--budget-mb", str(c["budget_mb"])]
    assert bench.plan_args(c, 3) == ["--k", "3"]
    assert bench.plan_args(bench.CONFIGS["cfg2"]) == ["--k", "1"]


def test_gpus_flag_launches_that_many_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself under
    torch.distributed.run with 2 ranks (gloo here; the launch-check hook stops
    after the ranks have joined); a WORLD_SIZE that disagrees with --gpus is
    refused."""
    import subprocess
    import sys

    env = dict(os.environ, LCL_BENCH_LAUNCH_CHECK="1", LCL_DIST_BACKEND="gloo",
               CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--config", "cfg1"], capture_output=True, text=True, env=env,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert lines == [{"launch_check": True, "n_gpus": 2, "ranks_joined": 2}]
    bad = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"],
                         capture_output=True, text=True, timeout=120,
                         env=dict(env, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0"))
    assert bad.returncode != 0 and "WORLD_SIZE=1" in bad.stderr
