"""Summaries committed under profiles/ from ncu output.

    python tools/ncu_summary.py full <report.ncu-rep> [label]    # --set full capture -> JSON
    python tools/ncu_summary.py launches <launches.csv> <title>  # launch list -> markdown

`full` prints, per captured kernel: duration, DRAM bytes, fp64-pipe and issue
utilisation, occupancy, registers, instructions and the top warp stalls.
`launches` aggregates a `ncu --metrics gpu__time_duration.sum,... --csv` log
(one row per metric per launch) into per-kernel totals and shares.
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

STALLS = "smsp__average_warps_issue_stalled_"


def _raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                         stdout=subprocess.PIPE).stdout.decode()
    rows = list(csv.reader(io.StringIO(out)))
    global _UNITS
    _UNITS = dict(zip(rows[0], rows[1]))
    return rows[0], rows[2:]


_UNITS = {}
_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
          "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def _f(r, hdr, name):
    """Value in base units: bytes, milliseconds, or as reported."""
    try:
        v = float(r[hdr.index(name)].replace(",", ""))
    except (ValueError, IndexError):
        return None
    return v * _SCALE.get(_UNITS.get(name, ""), 1.0)


def full(rep, label=""):
    hdr, rows = _raw(rep)
    out = []
    for r in rows:
        dur = _f(r, hdr, "gpu__time_duration.sum")
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith(STALLS) and h.endswith("_per_issue_active.ratio"):
                v = _f(r, hdr, h)
                if v:
                    stalls[h[len(STALLS):-len("_per_issue_active.ratio")]] = v
        tot = sum(stalls.values()) or 1.0
        top = dict(sorted(((k, round(100 * v / tot, 1)) for k, v in stalls.items()),
                          key=lambda kv: -kv[1])[:6])
        out.append({
            "kernel": r[hdr.index("Kernel Name")],
            "duration_ms": dur,
            "dram_read_GB": (_f(r, hdr, "dram__bytes_read.sum") or 0) / 1e9,
            "dram_write_GB": (_f(r, hdr, "dram__bytes_write.sum") or 0) / 1e9,
            "fp64_pipe_pct": _f(r, hdr, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": _f(r, hdr, "sm__inst_issued.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": _f(r, hdr, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "registers": _f(r, hdr, "launch__registers_per_thread"),
            "inst_executed": _f(r, hdr, "smsp__inst_executed.sum"),
            # fp64 arithmetic, thread level (a DFMA counts once)
            # (--set full carries the per-cycle rates: x the elapsed cycles of an SMSP)
            "fp64_thread_inst": {op: (_f(r, hdr, f"smsp__sass_thread_inst_executed_op_{op}_pred_on"
                                                 ".sum.per_cycle_elapsed") or 0.0)
                                 * (_f(r, hdr, "smsp__cycles_elapsed.avg") or 0.0)
                                 for op in ("dadd", "dmul", "dfma")},
            "fp64_pipe_warp_inst": _f(r, hdr, "sm__inst_executed_pipe_fp64.sum"),
            "top_stalls_pct": top,
        })
    return {"label": label, "report": rep, "kernels": out}


def launches(path, title):
    per = collections.defaultdict(lambda: {"n": 0, "ms": 0.0, "rd": 0.0, "wr": 0.0})
    text = open(path).read()
    text = text[text.index('"ID"'):] if '"ID"' in text else text
    for r in csv.DictReader(io.StringIO(text)):
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "")
        name = re.sub(r".*::", "", name)
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        d = per[(r["ID"], name)]
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["ms"] = v * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0,
                           "ms": 1.0, "second": 1e3, "s": 1e3}[unit]
        elif r["Metric Name"] == "dram__bytes_read.sum":
            d["rd"] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit.replace("B", "byte") if len(unit) <= 2 else unit, 1)
        elif r["Metric Name"] == "dram__bytes_write.sum":
            d["wr"] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit.replace("B", "byte") if len(unit) <= 2 else unit, 1)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for (_, name), d in per.items():
        a = agg[name]
        a[0] += 1
        a[1] += d["ms"]
        a[2] += d["rd"]
        a[3] += d["wr"]
    total = sum(a[1] for a in agg.values()) or 1.0
    lines = [f"# {title}", "",
             "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
             "--clock-control none` (cold-cache, serialised: compare shares, not absolute times).", "",
             "| kernel | launches | total ms | avg ms | DRAM GB / launch | share |", "|---|---|---|---|---|---|"]
    for name, (n, ms, rd, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {name} | {n} | {ms:.2f} | {ms / n:.4f} | {(rd + wr) / n / 1e9:.3f} | {100 * ms / total:.1f}% |")
    return "\n".join(lines) + "\n"


def fp64_ops(rep, cells, key, label, out_json):
    """Merge {key: fp64 instructions per cell-update} of the first captured kernel of
    `rep` (one Heun step over `cells` cells) into out_json (profiles/fp64_ops.json,
    read by bench.py for the fp64 roofline)."""
    k = full(rep)["kernels"][0]
    ops = sum(v for v in k["fp64_thread_inst"].values() if v)
    try:
        d = json.load(open(out_json))
    except (OSError, ValueError):
        d = {}
    d[key] = {"kernel": k["kernel"].split("(")[0], "fp64_ops_per_cell_update": ops / cells,
              "by_op_per_cell_update": {o: (v or 0) / cells for o, v in k["fp64_thread_inst"].items()},
              "fp64_pipe_warp_inst_per_cell_update": (k["fp64_pipe_warp_inst"] or 0) / cells,
              "inst_executed_per_cell_update": (k["inst_executed"] or 0) / cells,
              "duration_ms": k["duration_ms"], "fp64_pipe_pct": k["fp64_pipe_pct"],
              "issue_active_pct": k["issue_active_pct"], "registers": k["registers"],
              "top_stalls_pct": k["top_stalls_pct"], "source": label}
    json.dump(d, open(out_json, "w"), indent=1)
    return d[key]


if __name__ == "__main__":
    if sys.argv[1] == "fp64ops":
        print(json.dumps(fp64_ops(sys.argv[2], float(sys.argv[3]), sys.argv[4], sys.argv[5],
                                  sys.argv[6]), indent=1))
    elif sys.argv[1] == "full":
        print(json.dumps(full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""), indent=1))
    else:
        print(launches(sys.argv[2], sys.argv[3]))
