"""Attribute ncu warp-stall samples of a kernel to CUDA source lines.

    python tools/stall_lines.py <report.ncu-rep> '<name substring>@<mangled regex>' <cubin> [top]

Joins the report's per-SASS-instruction stall samples (--page source, SASS
view) with the cubin's line table (nvdisasm -g; build with -lineinfo).
"""
import collections
import csv
import io
import re
import subprocess
import sys


def sass_samples(rep, name_sub):
    """{offset: (samples, sass)} for the report section whose kernel name contains name_sub."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         stdout=subprocess.PIPE, check=True).stdout.decode()
    res, take, base, hdr = {}, False, None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "Kernel Name":
            take, base, hdr = name_sub in r[1], None, None
            continue
        if r[0] == "Address":
            hdr = r
            continue
        if not take or hdr is None:
            continue
        a = int(r[hdr.index("Address")], 16)
        base = a if base is None else base
        res[a - base] = (float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0),
                         r[hdr.index("Source")])
    return res


def line_table(cubin, fname_regex):
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], stdout=subprocess.PIPE, check=True).stdout.decode()
    cur_fn, cur_line, tab = None, None, {}
    for l in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", l)
        if m:
            cur_fn = m.group(1)
            continue
        m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', l)
        if m:
            cur_line = f"{m.group(1)}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m and cur_fn and re.search(fname_regex, cur_fn):
            tab[int(m.group(1), 16)] = cur_line
    return tab


def main(rep, kregex, cubin, top=40):
    # kregex: "<report name substring>@<mangled-name regex>", e.g.
    # "(bool)1, (bool)1@k_passILb1ELb1"
    sub, fre = kregex.split("@")
    samples = sass_samples(rep, sub)
    tab = line_table(cubin, fre)
    per = collections.Counter()
    tot = 0.0
    for a, (w, _) in samples.items():
        per[tab.get(a, "?")] += w
        tot += w
    print(f"total samples {tot:.0f}")
    for ln, w in per.most_common(top):
        print(f"  {ln:32s} {100 * w / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)
