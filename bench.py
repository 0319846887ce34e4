"""Benchmark: one encrypted Krum round of the Lancelot server path on B200.

A step = server step 3 + step 8 of the reference's run_round
(protocol.cpp:430-432, 492-493): build_distance_matrix(per_pair, lazy relin,
reduce_on_server) over all n clients, then masked_aggregate with the Krum
selection mask. Default workload = BASELINE.json configs[2] (cfg3), the
largest single-GPU config and the north star's named round: 20 clients,
11,173,962-parameter (ResNet-18) updates, CKKS N = 2^16 (342 chunks, 190
pairs, width 32768), lazy relinearisation and HOISTED rotations with the
unfold factor chosen dynamically as make_system does for HoistMode::dynamic_lp
(protocol.cpp:255-287): calibrate() timed on the device (lcl_calibrate), then
plan_unfold (distance.cpp:144-179) under the config's memory budget.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--config cfg3|cfg1|cfg2|cfg4] [--k K] [--budget-mb B]

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
with N ranks (one per GPU).

Our arm prints one JSON line (rank 0). `value` is device time per round with
inputs resident in HBM; `e2e` is the same round through the C-ABI entry
lcl_server_round_host with pinned host buffers (H2D of the clients and
selectors + D2H of the matrix and aggregate inside the timed region).
The reference arm (--impl reference) times the unmodified reference core
(oracle/_ref/ref_driver, built from /root/reference sources) on the host
cores for the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

# before any CUDA context: the host round's streams each get a hardware queue
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n clients, P params, N, k unfold | budget_mb (dynamic plan), rule, selected)
    "cfg1": dict(n=4, P=8192, N=8192, k=1),
    "cfg2": dict(n=10, P=272474, N=32768, k=1),
    # BASELINE configs[2]: "lazy relin + hoisted rotations". make_system's
    # dynamic plan picks the largest k the budget admits (plan_unfold's cost
    # falls with k whenever t_decompose < t_hoist); the reference's default
    # 1 GiB would pick k = 16 = 32767 rotation keys, which make_system
    # rejects (> 512, CapacityError), so the budget is part of the config:
    # 12 MiB = 3 fresh ciphertexts -> k = 3 (DESIGN.md §5 has the sweep).
    "cfg3": dict(n=20, P=11173962, N=65536, budget_mb=12.0),
    # BASELINE configs[3]: Multi-Krum, l = 25 selected (n - l > 2c + 2 for c = 10)
    "cfg4": dict(n=50, P=11173962, N=65536, k=1, rule="multi_krum", l=25),
}
METRIC = "Krum-round latency (ms) over encrypted updates"
DEFAULT_CONFIG = "cfg3"


def bit_ceil(x):
    return 1 << (x - 1).bit_length()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region through
    NVML (the library behind nvidia-smi) every 5 ms; falls back to polling
    the nvidia-smi CLI when NVML is unavailable."""

    REASONS = {  # nvmlClocksEventReason* bit masks
        "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index=0):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reason_mask)
        self._stop = threading.Event()
        self._ready = threading.Event()  # NVML initialised and sampling
        self._t = None

    def _run_nvml(self):
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((float(sm), float(mx), int(rs)))
            except Exception:
                pass
            self._ready.set()
            self._stop.wait(0.005)
        nv.nvmlShutdown()

    def _run_smi(self):
        q = "clocks.sm,clocks.max.sm,clocks_throttle_reasons.active"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip().split(",")
                self.samples.append((float(out[0]), float(out[1]), int(out[2].strip(), 16)))
            except Exception:
                pass
            self._ready.set()
            self._stop.wait(0.05)

    def _run(self):
        try:
            self._run_nvml()
        except Exception:
            self._run_smi()

    def __enter__(self):
        # NVML's first initialisation can take longer than a short timed
        # region: wait until the sampler runs, then keep only samples taken
        # from here on (the timed region)
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        self._ready.wait(timeout=10)
        self.samples.clear()
        return self

    def __exit__(self, *a):
        if not self.samples:  # a region shorter than one sampling period
            time.sleep(0.06)
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = sorted(s[0] for s in self.samples)
        reasons = sorted({n for s in self.samples for n, bit in self.REASONS.items() if s[2] & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples), "source": "nvml"}


# ------------------------------------------------------------------ reference arm
def reference_arm(args, cfg):
    """Times the reference's own CPU implementation (oracle/_ref/ref_driver,
    the unmodified reference core) on this host's cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    driver = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    line = {"impl": "reference", "metric": METRIC, "unit": "ms", "higher_is_better": False,
            "n_gpus": args.gpus, "config": workload(cfg, args.config, cfg.get("k"))}
    if not os.path.exists(driver):
        line["unavailable"] = "oracle/_ref/ref_driver not built (needs /root/reference at build time)"
        print(json.dumps(line))
        return
    cores = os.cpu_count() or 1
    env = dict(os.environ, LANCELOT_THREADS=str(cores))
    # The CPU reference needs no device warm-up; one untimed round absorbs
    # its first-call costs (Galois-table cache, thread pool) when the budget
    # allows, then as many timed rounds as fit (each a full round: cfg3 is
    # ~1.5 min on 16 cores). Inputs are uniform residues (data-oblivious
    # evaluator) so setup skips ~10 min of client encryption.
    reps = args.warmup + args.steps
    cmd = [driver, "bench", "--N", str(cfg["N"]), "--clients", str(cfg["n"]), "--dim",
           str(cfg["P"]), "--secure", "1", "--reps", str(reps), "--inputs", "uniform",
           "--rule", cfg.get("rule", "krum"),
           "--select", ",".join(str(i) for i in range(cfg.get("l", 1)))] + plan_args(cfg)
    t0 = time.time()
    proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, text=True, env=env)
    budget = args.ref_budget_s
    try:
        out, _ = proc.communicate(timeout=budget)
    except subprocess.TimeoutExpired:
        proc.kill()
        out, _ = proc.communicate()
    res = parse_partial_json(out)
    times = [r["distance_s"] + r["aggregate_s"] for r in res.get("reps", [])]
    warm = 1 if len(times) > 1 else 0
    timed = times[warm:]
    if not timed:
        line["unavailable"] = "reference run produced no timed repetition within the budget"
        print(json.dumps(line))
        return
    k = res.get("k", cfg.get("k"))
    line["config"] = workload(cfg, args.config, k)
    ms = 1000.0 * sum(timed) / len(timed)
    sample = (f"full {args.config} round (build_distance_matrix per_pair lazy reduce, k={k} + "
              f"masked_aggregate {cfg.get('rule', 'krum')}) x {len(timed)} timed reps after {warm} "
              f"untimed; uniform-residue inputs; setup (keygen + calibrate + inputs) "
              f"{res.get('setup_s', 0):.1f}s excluded; wall {time.time() - t0:.0f}s")
    line.update({"value": ms, "steps": len(timed), "warmup": warm, "ms_per_step": ms,
                 "scaling": "replicas", "vs_baseline": None, "dtype": "u64",
                 "data": "synthetic: uniform residues mod each q_i for client chunks and selectors, "
                         "keys from the reference's generate_keys",
                 "plan": plan_record(res, cfg, "reference calibrate() on the host CPU"),
                 "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "reference",
                                  "sample": sample},
                 "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    print(json.dumps(line))


def plan_args(cfg, k=None):
    """ref_driver options for the config's hoisting plan: a fixed k, or
    calibrate + plan_unfold under the memory budget (k = 0)."""
    if k is not None:
        return ["--k", str(k)]
    if "budget_mb" in cfg:
        return ["--k", "0", "--budget-mb", str(cfg["budget_mb"])]
    return ["--k", str(cfg["k"])]


def plan_record(res, cfg, source):
    if "budget_mb" not in cfg:
        return {"hoisting": "fixed", "k": res.get("k", cfg.get("k"))}
    return {"hoisting": "dynamic_lp", "memory_budget_mb": cfg["budget_mb"], "k": res.get("k"),
            "t_hoist_s": res.get("t_hoist"), "t_decompose_s": res.get("t_decompose"),
            "m_cipher": res.get("m_cipher"), "calibrated_on": source}


def parse_partial_json(out):
    out = out.strip()
    try:
        return json.loads(out)
    except Exception:
        pass
    # truncated run: close the list
    i = out.rfind("}")
    if i < 0:
        return {}
    try:
        return json.loads(out[: i + 1] + "]}")
    except Exception:
        return {}


def workload(cfg, name, k):
    N = cfg["N"]
    slots = N // 2
    C = (cfg["P"] + slots - 1) // slots
    d = {"workload": f"{name}: encrypted Krum round, {cfg['n']} clients x {cfg['P']} params, "
                     f"CKKS N=2^{N.bit_length() - 1}",
         "clients": cfg["n"], "params": cfg["P"], "ring_degree": N, "chunks": C,
         "pairs": cfg["n"] * (cfg["n"] - 1) // 2, "reduce_width": bit_ceil(min(cfg["P"], slots)),
         "unfold_k": k, "hoisting": "dynamic_lp" if "budget_mb" in cfg else "fixed",
         "lazy_relin": True, "rule": cfg.get("rule", "krum"),
         "selected": cfg.get("l", 1),
         "l2": "flushed between steps (256 MiB write) and client data > L2"}
    if "budget_mb" in cfg:
        d["memory_budget_mb"] = cfg["budget_mb"]
    return d


# ------------------------------------------------------------------ cpu baseline
def cpu_baseline(cfg, name, budget_s, k):
    """The unmodified reference (oracle/_ref) timed for one full round of the
    same workload and plan (k) on all host cores, rank 0 at N = 1."""
    driver = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    cores = os.cpu_count() or 1
    if not os.path.exists(driver):
        return {"value": None, "unit": "ms", "cores": cores, "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    env = dict(os.environ, LANCELOT_THREADS=str(cores))
    cmd = [driver, "bench", "--N", str(cfg["N"]), "--clients", str(cfg["n"]), "--dim",
           str(cfg["P"]), "--secure", "1", "--reps", "1", "--inputs", "uniform",
           "--rule", cfg.get("rule", "krum"),
           "--select", ",".join(str(i) for i in range(cfg.get("l", 1)))] + plan_args(cfg, k)
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=budget_s).stdout
        res = json.loads(out)
        r = res["reps"][0]
        ms = 1000.0 * (r["distance_s"] + r["aggregate_s"])
        return {"value": ms, "unit": "ms", "cores": cores, "kind": "reference",
                "sample": f"one full {name} round (k={k}) on the unmodified reference core "
                          f"(distance {r['distance_s']:.2f}s + aggregate {r['aggregate_s']:.2f}s), "
                          f"LANCELOT_THREADS={cores}, uniform-residue inputs; setup "
                          f"{res['setup_s']:.1f}s excluded"}
    except Exception as e:  # noqa: BLE001
        return {"value": None, "unit": "ms", "cores": cores, "kind": "reference",
                "sample": f"failed: {e}"[:200]}


# ------------------------------------------------------------------ our arm
def our_arm(args, cfg):
    global TRAFFIC_CONFIG
    TRAFFIC_CONFIG = args.config
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2408_06197_b200.lancelot as L

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # LCL_DIST_BACKEND / LCL_ONE_DEVICE: a test hook that runs the
        # multi-rank orchestration as N ranks on ONE GPU over gloo (no N-GPU
        # number is ever reported from it; see tools/gpu_multirank_smoke.sh)
        dist.init_process_group(os.environ.get("LCL_DIST_BACKEND", "nccl"))
    if os.environ.get("LCL_BENCH_LAUNCH_CHECK") == "1":
        # CPU test hook (tests/test_bench_contract.py): the rank plumbing of
        # --gpus N only -- every rank joins, rank 0 reports the world size
        t = torch.ones(1)
        if world > 1:
            dist.all_reduce(t)
            dist.destroy_process_group()
        if rank == 0:
            print(json.dumps({"launch_check": True, "n_gpus": world, "ranks_joined": int(t.item())}))
        return
    if os.environ.get("LCL_ONE_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    N, n = cfg["N"], cfg["n"]
    slots = N // 2
    Cc = (cfg["P"] + slots - 1) // slots
    width = bit_ceil(min(cfg["P"], slots))
    ctx = L.CkksContext(L.CkksParams(ring_degree=N), device=local)
    stream = torch.cuda.Stream(device=dev)
    ctx.set_stream(stream)
    m = ctx.full
    primes = ctx.primes + [ctx.special]
    g = torch.Generator(device=dev)
    g.manual_seed(1234)  # identical (replicated) inputs on every rank

    def residues(*shape, rows_last=2, row_primes=None):
        t = torch.empty(shape, dtype=torch.int64, device=dev)
        for r, q in enumerate(row_primes):
            sl = [slice(None)] * len(shape)
            sl[-rows_last] = r
            t[tuple(sl)] = torch.randint(0, q, shape[:-rows_last] + shape[-rows_last + 1:],
                                         generator=g, device=dev, dtype=torch.int64)
        return t

    # keys: [full][2][full+1][N], uniform residues per row prime (data-oblivious kernels)
    def key():
        return L.to_host(residues(m, 2, m + 1, N, row_primes=primes))

    # the hoisting plan: fixed k, or make_system's dynamic_lp plan from a
    # device calibration (probe keys {1, 2}, a fresh ciphertext) under the
    # config's memory budget; rank 0's plan is broadcast so ranks agree
    plan = {"hoisting": "fixed", "k": cfg.get("k")}
    if "k" in cfg:
        k = cfg["k"]
    else:
        probe = L.RotationKeySet({1: key(), 2: key()})
        fresh = L.Ciphertext(residues(2, m, N, row_primes=primes[:m]), ctx.scale())
        with torch.cuda.stream(stream):
            cal = L.calibrate(ctx, probe, fresh)
        hp = L.plan_unfold(cal.t_hoist, cal.t_decompose, cal.m_cipher,
                           cfg["budget_mb"] * 1048576.0, width)
        k = hp.k
        if world > 1:
            kt = torch.tensor([k], device=dev)
            dist.broadcast(kt, 0)
            k = int(kt.item())
        plan = {"hoisting": "dynamic_lp", "memory_budget_mb": cfg["budget_mb"], "k": k,
                "t_hoist_s": cal.t_hoist, "t_decompose_s": cal.t_decompose,
                "m_cipher": cal.m_cipher, "plan_cost_s": hp.cost,
                "calibrated_on": "device (lcl_calibrate: median of 11 CUDA-event-timed "
                                 "hoisted_rotations calls, batch 1)"}
    rk = L.RelinKey(key())
    steps = L.slot_reduce_steps(width, k)
    keys = L.RotationKeySet({s: key() for s in steps})
    ctx.use_relin_key(rk)
    ctx.use_rotation_keys(keys, steps)
    # one GPU holds every chunk; with N > 1 GPUs rank r holds only its chunk
    # slice of every client (chunk-sharded round)
    from paper_2408_06197_b200.sharded import shard_range
    cr0, cr1 = shard_range(Cc, world, rank)
    clients = residues(n, cr1 - cr0, 2, m, N, row_primes=primes[:m])
    sel = residues(n, 2, m, N, row_primes=primes[:m])
    npairs = n * (n - 1) // 2
    d_dist = torch.empty(npairs, 2, m - 1, N, dtype=torch.int64, device=dev)
    l_sel = cfg.get("l", 1)
    average = cfg.get("rule") == "multi_krum" and l_sel > 1
    d_agg = torch.empty(Cc, 2, m - 2 if average else m - 1, N, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    scale = ctx.scale()
    osc = C.c_double()
    lib = L.lib()

    if world == 1:
        def step():  # run_round steps 3 + 8: distance matrix and (concurrently) the aggregate
            L._check(lib.lcl_server_round(ctx.h, L._ptr(clients), L._ptr(sel), n, Cc, width, k, l_sel,
                                          1 if average else 0, L._ptr(d_dist), L._ptr(d_agg)))
            return d_dist, d_agg
    else:
        # chunk-sharded: partial ternaries of all pairs over the local chunks,
        # integer reduce_scatter (NCCL / NVLink), pair-sharded key-switch
        # chains, local aggregate chunks, all-gather of both results
        from paper_2408_06197_b200.sharded import chunk_sharded_server_round, cuda_chunk_shard_fns
        fpart, ffin, fch, du, au = cuda_chunk_shard_fns(ctx, clients, sel, n, cr1 - cr0, scale,
                                                        scale, width, k, l=l_sel, average=average)

        def step():
            return chunk_sharded_server_round(npairs, Cc, du, au, fpart, ffin, fch)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        stream.synchronize()
        # CUDA graph of the whole round (single GPU): after warm-up every
        # workspace exists and the Krum round has no host synchronisation,
        # so the ~140 launches are captured once and replayed.
        graph = None
        launches_per_step = None
        if world == 1 and not args.no_graph:
            l0 = ctx.launch_count()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                step()
            launches_per_step = ctx.launch_count() - l0
            graph.replay()
            stream.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        launches0 = ctx.launch_count()
        total_ms = 0.0
        with ClockSampler(local) as clk:
            for _ in range(args.steps):
                flush.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                if graph is not None:
                    graph.replay()
                else:
                    step()
                b.record(stream)
                b.synchronize()
                total_ms += a.elapsed_time(b)
        launches = ctx.launch_count() - launches0
        if graph is not None:
            launches = launches_per_step * args.steps
        torch.cuda.synchronize()
    ms = total_ms / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- end to end with pinned host buffers: through the C-ABI host entry
    # (lcl_server_round_host) on one GPU; with N > 1 GPUs, H2D of each rank's
    # chunk slice and the selectors, the sharded round and D2H of the gathered
    # outputs on every rank.
    def measure_e2e():
        h_dist = torch.empty(d_dist.shape, dtype=torch.int64, pin_memory=True)
        h_agg = torch.empty(d_agg.shape, dtype=torch.int64, pin_memory=True)
        if world == 1 and not args.e2e_words:
            # the server's real input: the clients' and the KGC's LCLT blobs
            # (CkksContext::serialize bytes, run_round step 3 deserializes them,
            # protocol.cpp:419-432), in pinned host memory at a 64-byte stride
            bb = ctx.blob_bytes()
            stride = (bb + 63) // 64 * 64
            h_cb = torch.empty((n * Cc, stride), dtype=torch.uint8, pin_memory=True)
            h_sb = torch.empty((n, stride), dtype=torch.uint8, pin_memory=True)
            with torch.cuda.stream(stream):
                for i in range(n):
                    L._check(lib.lcl_serialize(ctx.h, L._ptr(clients[i]), Cc, m, scale,
                                               C.c_void_p(h_cb[i * Cc].data_ptr()), stride))
                L._check(lib.lcl_serialize(ctx.h, L._ptr(sel), n, m, scale,
                                           C.c_void_p(h_sb.data_ptr()), stride))
            dsc, asc = C.c_double(), C.c_double()

            def e2e_step():
                L._check(lib.lcl_server_round_lclt(
                    ctx.h, C.c_void_p(h_cb.data_ptr()), C.c_void_p(h_sb.data_ptr()), bb, stride, n,
                    Cc, width, k, l_sel, 1 if average else 0, C.c_void_p(h_dist.data_ptr()),
                    C.c_void_p(h_agg.data_ptr()), C.byref(dsc), C.byref(asc)))
            h2d = h_cb.numel() + h_sb.numel()
            ingest = (f"LCLT blobs ({bb} B each at a {stride} B stride, pinned) through "
                      "lcl_server_round_lclt: header checks on the host, verbatim H2D, device "
                      "unpack + residue checks inside the overlapped pipeline")
        else:
            h_clients = torch.empty(clients.shape, dtype=torch.int64, pin_memory=True)
            h_clients.copy_(clients.cpu())
            h_sel = torch.empty(sel.shape, dtype=torch.int64, pin_memory=True)
            h_sel.copy_(sel.cpu())
            h2d = (h_clients.numel() + h_sel.numel()) * 8
            ingest = "limb-major u64 words (pinned) through lcl_server_round_host"

        def e2e_step_words():
            if world == 1:
                L._check(lib.lcl_server_round_host(ctx.h, C.c_void_p(h_clients.data_ptr()),
                                                   C.c_void_p(h_sel.data_ptr()), n, Cc, scale, width,
                                                   k, l_sel, 1 if average else 0,
                                                   C.c_void_p(h_dist.data_ptr()),
                                                   C.c_void_p(h_agg.data_ptr())))
                return
            clients.copy_(h_clients, non_blocking=True)
            sel.copy_(h_sel, non_blocking=True)
            dd, aa = step()
            h_dist.copy_(dd, non_blocking=True)
            h_agg.copy_(aa, non_blocking=True)

        if world > 1 or args.e2e_words:
            e2e_step = e2e_step_words

        with torch.cuda.stream(stream):
            e2e_step()
            e2e_step()
        e2e_ms = 0.0
        e2e_steps = max(3, min(args.steps, 10))
        with torch.cuda.stream(stream):
            for _ in range(e2e_steps):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                e2e_step()
                b.record(stream)
                b.synchronize()
                e2e_ms += a.elapsed_time(b)
        e2e_ms /= e2e_steps
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        d2h = (h_dist.numel() + h_agg.numel()) * 8
        return e2e_ms, h2d, d2h, ingest

    e2e = None
    if not args.no_e2e:
        e2e_ms, h2d, d2h, ingest = measure_e2e()
        e2e = {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ingest": ingest}

    # ---- per-kernel breakdown of one profiled round (CUDA events per launch)
    with torch.cuda.stream(stream):
        prof = profile_round(ctx, step, stream, N, m, npairs, cr1 - cr0, width, n)

    if rank == 0:
        cpu = (cpu_baseline(cfg, args.config, args.cpu_budget_s, k)
               if world == 1 and not args.no_cpu else None)
        line = {
            "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "parallelism": (f"chunks sharded over {world} GPUs (partial ternaries joined by one NCCL "
                            f"reduce_scatter), pair chains sharded, all-gather") if world > 1 else "1 GPU",
            "data": "synthetic: uniform residues mod each q_i for ciphertexts, selectors and keys "
                    "(every kernel is data-oblivious; bit-exactness is proven by tests/)",
            "config": workload(cfg, args.config, k),
            "plan": plan,
            "clocks": clk.summary(),
            "e2e": e2e if e2e is not None else {"value": None, "skipped": "--no-e2e"},
            "gpu_launches": int(launches // max(1, args.steps)),
            "cuda_graph": graph is not None,
            "roofline": prof.get("roofline"),
            "roofline_int": prof.get("roofline_int"),
            "roofline_fp64": prof.get("roofline_fp64"),
            "kernels": prof.get("kernels"),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def profile_round(ctx, step, stream, N, m, npairs, Cc, width, n):
    """Times every launch of one round with CUDA events on the context's
    stream (lcl_profile_begin/end) and returns the per-kernel totals plus the
    rooflines of the top kernel: HBM (algorithmic bytes / time vs the measured
    copy bandwidth) and integer (algorithmic butterflies / time vs the
    measured butterfly peak of lcl_peak_butterflies)."""
    import ctypes as C
    import json as _json

    import paper_2408_06197_b200.lancelot as L
    lib = L.lib()
    step()
    stream.synchronize()
    L._check(lib.lcl_profile_begin(ctx.h))
    step()
    buf = C.create_string_buffer(1 << 20)
    L._check(lib.lcl_profile_end(ctx.h, buf, len(buf)))
    rows = _json.loads(buf.value.decode())
    peak = C.c_double()
    L._check(lib.lcl_peak_butterflies(ctx.h, C.byref(peak)))
    peak_f = C.c_double()
    L._check(lib.lcl_peak_butterflies_f64(ctx.h, C.byref(peak_f)))
    peaks = load_peaks()
    kernels = sorted(rows, key=lambda r: -r["ms"])
    total = sum(k["ms"] for k in kernels)
    for k in kernels:
        s = k["ms"] * 1e-3
        k["hbm_gbs"] = k["bytes"] / s / 1e9
        k["gbfly_s"] = k["bfly"] / s / 1e9 if k["bfly"] else None
        k["share"] = k["ms"] / total
    top = kernels[0]
    avg_s = top["ms"] / top["launches"] * 1e-3
    achieved = top["bytes"] / top["launches"] / avg_s / 1e9
    roof = {"bound": "hbm", "kernel": top["name"], "achieved": achieved,
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
            "traffic": None, "peak_source": peaks["source"],
            "bytes_per_launch": top["bytes"] / top["launches"],
            "avg_launch_ms": top["ms"] / top["launches"], "share_of_round": top["share"]}
    tr = traffic_for(top["name"], roof["bytes_per_launch"])
    if tr:
        roof["traffic"] = tr["dram_bytes_per_launch"]
        roof["traffic_over_algorithmic"] = tr["ratio"]
        roof["traffic_source"] = tr["source"]
    int_roof = None
    if top["bfly"]:
        ach = top["bfly"] / top["launches"] / avg_s / 1e9
        int_roof = {"bound": "int (64-bit Shoup butterflies)", "kernel": top["name"],
                    "achieved": ach, "peak": peak.value, "unit": "Gbfly/s",
                    "frac": ach / peak.value,
                    "peak_fp64": peak_f.value, "frac_fp64": ach / peak_f.value,
                    "peak_source": "measured live: lcl_peak_butterflies / _f64 (register-resident "
                                   "independent CT butterflies of each field, all SMs); q-chain "
                                   "rows run on the FP64 pipe, the special prime on the integer "
                                   "pipe, so the kernel's bound lies between the two"}
    # the pair accumulation runs on the FP64 pipe (q-chain < 2^44): 17 FP64
    # ops per pair-slot-chunk (2 DADD + 3 x (2 DFMA + 2 DADD + 1 DFMA)) against
    # 64 ops/clk/SM at the SM clock the round ran at
    fp64_roof = None
    pk = next((k for k in kernels if k["name"] == "pair_accumulate"), None)
    if pk is not None:
        import torch
        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        ops = 17.0 * npairs * Cc * m * N
        ach = ops / (pk["ms"] * 1e-3) / 1e12
        pk_peak = 64.0 * sms * 1.965e9 / 1e12
        fp64_roof = {"bound": "fp64 pipe", "kernel": "pair_accumulate", "achieved": ach,
                     "peak": pk_peak, "unit": "Tops/s", "frac": ach / pk_peak,
                     "ops": ops, "peak_source": f"64 FP64 ops/clk/SM x {sms} SMs x 1965 MHz "
                     "(4.27 pair-slots/clk/SM = 93% of it reached by tools/microbench/pair_forms.cu)"}
    if top["name"] == "pair_accumulate" and fp64_roof is not None:
        # the top kernel is bound by the FP64 pipe, not HBM (its traffic is
        # the compulsory client bytes, ~19 % of HBM at cfg3): report it against
        # that pipe, keep the HBM view beside it
        hbm_view = roof
        roof = dict(fp64_roof)
        roof.update({"bound": "fp64", "traffic": hbm_view.get("traffic"),
                     "avg_launch_ms": hbm_view["avg_launch_ms"],
                     "share_of_round": hbm_view["share_of_round"], "hbm_view": hbm_view})
    return {"roofline": roof, "roofline_int": int_roof, "roofline_fp64": fp64_roof,
            "kernels": kernels[:12], "peak_gbfly_s": peak.value, "peak_gbfly_s_fp64": peak_f.value}


TRAFFIC_CONFIG = None  # set by our_arm: the config whose ncu traffic file applies


def traffic_for(kernel, algorithmic_bytes):
    """DRAM bytes per launch of `kernel` from the committed ncu capture of one
    round of this config (profiles/r01_traffic_<cfg>.json, tools/ncu_traffic.py),
    or None when no capture exists."""
    p = os.path.join(ROOT, "profiles", f"r02_traffic_{TRAFFIC_CONFIG}.json")
    if not os.path.exists(p):
        p = os.path.join(ROOT, "profiles", f"r01_traffic_{TRAFFIC_CONFIG}.json")
    try:
        with open(p) as f:
            k = json.load(f)["kernels"][kernel]
        return {"dram_bytes_per_launch": k["dram_bytes_per_launch"],
                "algorithmic_bytes_per_launch": algorithmic_bytes,
                "ratio": k["dram_bytes_per_launch"] / algorithmic_bytes,
                "source": os.path.relpath(p, ROOT)}
    except Exception:
        return None


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def self_launch(args):
    """--gpus N > 1 outside torchrun: re-run this script under
    torch.distributed.run with N ranks on this node (127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the round eagerly")
    ap.add_argument("--no-e2e", action="store_true",
                    help="skip the host-buffer round (cfg4: its 72 GB of pinned client data "
                         "exceed what a host should pin)")
    ap.add_argument("--cpu-budget-s", type=float, default=400.0)
    ap.add_argument("--ref-budget-s", type=float, default=250.0)
    ap.add_argument("--k", type=int, default=None, help="fixed unfold factor (overrides the plan)")
    ap.add_argument("--e2e-words", action="store_true",
                    help="end-to-end from limb-major words (lcl_server_round_host) instead of "
                         "LCLT blobs")
    ap.add_argument("--budget-mb", type=float, default=None,
                    help="memory budget of the dynamic plan (overrides the config's)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = dict(CONFIGS[args.config])
    if args.k:
        cfg.pop("budget_mb", None)
        cfg["k"] = args.k
    elif args.budget_mb:
        cfg.pop("k", None)
        cfg["budget_mb"] = args.budget_mb
    world = os.environ.get("WORLD_SIZE")
    if args.impl == "reference":
        reference_arm(args, cfg)
        return 0
    if world is None and args.gpus > 1:
        return self_launch(args)
    if world is not None and int(world) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    our_arm(args, cfg)
    return 0


if __name__ == "__main__":
    sys.exit(main())
