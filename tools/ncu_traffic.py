"""Per-kernel DRAM traffic of one server round from an ncu capture, keyed by
the names bench.py's per-launch profile uses, for the `roofline.traffic`
field (dram__bytes_read.sum + dram__bytes_write.sum per launch).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none --csv --log-file gpurun_out/traffic_cfg2.csv \
        python tools/one_round.py --config cfg2
    python tools/ncu_traffic.py gpurun_out/traffic_cfg2.csv > profiles/r01_traffic_cfg2.json

modup_ip_blk launches with and without the Galois permutation share one
template; they are told apart by their order in the round (the relinearize
ModUp precedes the slot_reduce rotations), so here both map to the
per-launch average of the template, reported under both names.
"""
import csv
import json
import re
import sys
from collections import defaultdict


def bench_name(kernel):
    k = kernel.split("(")[0].replace("void ", "").replace("lcl::", "").strip()
    base = k.split("<")[0]
    if base == "ntt_blk_fwd":
        if "DivRoundInvStore" in k:
            return "ntt_blk_fwd<divround+inv>"
        return "ntt_blk_fwd<divround>" if "DivRoundStore" in k else "ntt_blk_fwd"
    if base.startswith("pair_accumulate"):
        return "pair_accumulate"
    if base == "aggregate_stream":
        return "aggregate_tensor"
    return base


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    iid = hdr.index("ID")
    per = defaultdict(dict)
    for r in rows[start + 1:]:
        if len(r) <= iv:
            continue
        v = float(r[iv].replace(",", ""))
        per[(int(r[iid]), r[ik])][r[im]] = v
    acc = defaultdict(lambda: [0, 0.0, 0.0])
    for (lid, k), mets in per.items():
        a = acc[bench_name(k)]
        a[0] += 1
        a[1] += mets.get("dram__bytes_read.sum", 0) + mets.get("dram__bytes_write.sum", 0)
        a[2] += mets.get("gpu__time_duration.sum", 0)
    out = {name: {"launches": n, "dram_bytes_per_launch": b / n, "ncu_ns_per_launch": t / n}
           for name, (n, b, t) in acc.items()}
    if "modup_ip_blk" in out:
        out["modup_ip_blk<perm>"] = out["modup_ip_blk"]
    json.dump({"source": sys.argv[1], "units": "bytes (dram read + write), ns (ncu, serialised)",
               "kernels": out}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
