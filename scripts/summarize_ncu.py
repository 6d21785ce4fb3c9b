"""Summarise ncu output into profiles/ (run here, on the CPU box).

    python scripts/summarize_ncu.py --launches gpurun_out/launches_r1.csv \
        --report gpurun_out/prof_r1.ncu-rep --config llama8b --tag r1

Writes profiles/<tag>_launches.md (per-kernel share of one step from the
serialised, cold-cache launch list), profiles/<tag>_ncu_full.md (key metrics
of the --set full capture) and merges per-kernel DRAM traffic into
profiles/ncu_traffic.json (bench.py reads it for roofline.traffic).
"""

import argparse
import csv
import io
import json
import os
import re
import subprocess
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLASS = OrderedDict([
    ("scaled_prep_kernel", "bwd_g"), ("target_dot_kernel", "gather"),
    ("EpiLse", "fwd_gemm"), ("EpiG", "bwd_g"), ("EpiDH", "bwd_dh"), ("EpiDW", "bwd_dw"),
    ("prep_kernel", "prep"), ("gather_kernel", "gather"), ("combine_kernel", "combine"),
    ("combine_rows_kernel", "combine"), ("loss_reduce_kernel", "combine"), ("fixup_g_kernel", "bwd_g"), ("fixup_q_kernel", "bwd_g"),
    ("finalize_dh_kernel", "finalize"), ("reduce_dh_kernel", "finalize"), ("EpiAdamW", "bwd_dw"),
])


def classify(name):
    for k, v in CLASS.items():
        if k in name:
            return v
    return None


def read_csv_after_header(path):
    txt = open(path).read()
    i = txt.index('"ID"')
    return list(csv.DictReader(io.StringIO(txt[i:])))


def launches(path, steps):
    rows = read_csv_after_header(path)
    per = OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        c = classify(r["Kernel Name"])
        if c is None:
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
        t = float(r["Metric Value"].replace(",", "")) * scale
        per.setdefault(c, []).append(t)
    return per


def full_metrics(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__cycles_elapsed.avg.per_second", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg", "sm__cycles_elapsed.max"]
    res = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        d = {"kernel": name, "class": classify(name)}
        for w in want:
            if w in hdr:
                i = hdr.index(w)
                d[w] = (r[i], units[i])
        res.append(d)
    return res


def to_bytes(v, u):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    ap.add_argument("--config", default="llama8b")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--steps", type=int, default=3, help="fwd+bwd steps in the launch list (warmup + timed)")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if a.launches:
        per = launches(a.launches, a.steps)
        tot = sum(sum(v) for v in per.values())
        lines = [f"# {a.tag}: ncu launch list ({a.config}), `gpu__time_duration.sum --clock-control none`",
                 "", "Serialised, cold-cache launches; compare shares, not absolutes.", "",
                 "| kernel class | launches | total us | mean us/launch | share of LCE device time |",
                 "|---|---|---|---|---|"]
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| {k} | {len(v)} | {sum(v):.1f} | {sum(v) / len(v):.1f} | {sum(v) / tot:.3f} |")
        open(os.path.join(ROOT, "profiles", f"{a.tag}_launches.md"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
    if a.report:
        res = full_metrics(a.report)
        lines = [f"# {a.tag}: ncu --set full ({a.config}), one launch per kernel class of one row chunk", "",
                 "| kernel | class | duration | DRAM read | DRAM write | tensor pipe active | SM active / elapsed cycles | SM clock | L2 thr. | DRAM thr. | regs |",
                 "|---|---|---|---|---|---|---|---|---|---|---|"]
        tj_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        tj = json.load(open(tj_path)) if os.path.exists(tj_path) else {}
        cfg = tj.setdefault(a.config, {})
        run_max = {}
        for d in res:
            g = lambda k: "%s %s" % d[k] if k in d else "-"  # noqa: E731
            short = re.sub(r"\(.*", "", d["kernel"]).replace("void ", "")
            lines.append(f"| `{short}` | {d['class']} | {g('gpu__time_duration.sum')} | {g('dram__bytes_read.sum')} | "
                         f"{g('dram__bytes_write.sum')} | {g('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active')} | "
                         f"{d.get('sm__cycles_active.avg', ('-',))[0]} / {d.get('sm__cycles_elapsed.max', ('-',))[0]} | "
                         f"{g('sm__cycles_elapsed.avg.per_second')} | {g('lts__throughput.avg.pct_of_peak_sustained_elapsed')} | "
                         f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')} | {g('launch__registers_per_thread')} |")
            if d["class"] and "dram__bytes_read.sum" in d:
                b = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
                # a class may appear twice (the scaled-q path's gated, usually empty
                # re-forward is an EpiLse launch too): keep the real launch's bytes
                seen = run_max.get(d["class"], 0.0)
                run_max[d["class"]] = max(seen, b)
                cfg[d["class"]] = run_max[d["class"]]
        tj[a.config] = cfg
        json.dump(tj, open(tj_path, "w"), indent=1)
        open(os.path.join(ROOT, "profiles", f"{a.tag}_ncu_full.md"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))


if __name__ == "__main__":
    main()
