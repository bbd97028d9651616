"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch) by
kernel, and optionally write profiles/traffic.json for bench.py's roofline.

  python tools/ncu_launches.py gpurun_out/r01/launches_bench.csv [--traffic profiles/traffic.json [--workload C2]]
"""
import collections
import csv
import json
import re
import sys


def short(name):
    n = name.split("(")[0].replace("void ", "")
    n = re.sub(r"gfwa::<unnamed>::", "", n)
    return n[:70]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h = [r for r in rows if r and r[0] == "ID"][0]
    data = [r for r in rows if len(r) == len(h) and r[0] != "ID"]
    per = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in data:
        per[short(r[h.index("Kernel Name")])][r[h.index("Metric Name")]].append(
            float(r[h.index("Metric Value")].replace(",", "")))
    out = {}
    print(f"{'kernel':70s} {'n':>4s} {'us/launch':>10s} {'rd MB':>9s} {'wr MB':>9s} {'GB/s':>8s}")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
        n = len(v["gpu__time_duration.sum"])
        t = sum(v["gpu__time_duration.sum"]) / n
        rd = sum(v.get("dram__bytes_read.sum", [0])) / n
        wr = sum(v.get("dram__bytes_write.sum", [0])) / n
        out[k] = {"n": n, "ns": t, "dram_read": rd, "dram_write": wr}
        print(f"{k:70s} {n:4d} {t / 1e3:10.2f} {rd / 1e6:9.2f} {wr / 1e6:9.2f} {(rd + wr) / t:8.1f}")
    if "--traffic" in sys.argv:
        path = sys.argv[sys.argv.index("--traffic") + 1]
        call = {"fwd": ["fwd_tc_kernel"], "bwd": ["bwd_tc_pre", "bwd_tc_kernel", "bwd_tc_post"],
                "bwd_main": ["bwd_tc_kernel"]}
        tr = {kind: sum(out[k]["dram_read"] + out[k]["dram_write"] for k in out if any(k.startswith(x) for x in ks))
              for kind, ks in call.items()}
        tr = {k: int(v) for k, v in tr.items() if v}
        tr["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch: fwd = fwd_tc_kernel, bwd = the "
                       "gfwa_bwd call (pre + main + post), bwd_main = bwd_tc_kernel alone; from " + sys.argv[1])
        wl = sys.argv[sys.argv.index("--workload") + 1] if "--workload" in sys.argv else "C2"
        try:
            allt = json.load(open(path))
        except Exception:
            allt = {}
        allt = {k: v for k, v in allt.items() if isinstance(v, dict)}  # per-workload entries only
        allt[wl] = tr
        json.dump(allt, open(path, "w"), indent=1)
        print("wrote", path, tr)


if __name__ == "__main__":
    main()
