"""Static SASS mix of a kernel's main loop (the longest backward branch).

    python tools/sass_mix.py <lib.so> <kernel-name-regex> [top]
"""
import collections
import re
import subprocess
import sys


def main(so, pat, top=40):
    out = subprocess.run(["cuobjdump", "-sass", so], check=True, stdout=subprocess.PIPE).stdout.decode()
    cur, funcs = None, {}
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
        if cur and m:
            funcs[cur].append((int(m.group(1), 16), m.group(2).strip()))
    for name, ins in funcs.items():
        if not re.search(pat, name):
            continue
        best = None
        for a, b in ins:
            # the main loop closes with a predicated backward branch; the
            # unconditional ones return from out-of-line slow paths
            m = re.search(r"^@!?U?P\w+ BRA (?:`\()?.*?0x([0-9a-f]+)", b)
            if m and int(m.group(1), 16) < a:
                t = int(m.group(1), 16)
                if best is None or a - t > best[1] - best[0]:
                    best = (t, a)
        body = [b for a, b in ins if best and best[0] <= a <= best[1]]
        cnt = collections.Counter()
        for b in body:
            t = b.split()
            cnt[t[1] if t[0].startswith("@") else t[0]] += 1
        print(name, "total", len(ins), "loop", len(body))
        for op, n in cnt.most_common(top):
            print("   %-28s %4d" % (op, n))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
