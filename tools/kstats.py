"""Summarise ptxas -v logs (registers/spills) and SASS opcode counts of the built kernels."""
import collections
import re
import subprocess
import sys


def ptxas(paths):
    cur = None
    for p in paths:
        for line in open(p):
            m = re.search(r"Compiling entry function '(\S+)'", line)
            if m:
                cur = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
                cur = re.sub(r"adct::\(anonymous namespace\)::", "", cur)
                cur = re.sub(r"\(.*", "", cur)
            m = re.search(r"Used (\d+) registers", line)
            if m and cur:
                sp = re.search(r"(\d+) bytes spill stores", prev) if prev else None
                print(f"{int(m.group(1)):4d} regs  spill={sp.group(1) if sp else '?':>4}  {cur}")
            prev = line


def sass(so, pattern):
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    fn, counts = None, collections.Counter()
    res = []
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if fn:
                res.append((fn, counts))
            fn, counts = m.group(1), collections.Counter()
            continue
        m = re.search(r"/\*[0-9a-f]{4,5}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]+)", line)
        if m and fn:
            counts[m.group(1)] += 1
    if fn:
        res.append((fn, counts))
    for fn, c in res:
        name = subprocess.run(["c++filt"], input=fn, capture_output=True, text=True).stdout.strip()
        if re.search(pattern, name):
            tot = sum(v for k, v in c.items() if k not in ("NOP",))
            print(re.sub(r"adct::\(anonymous namespace\)::", "", name)[:110])
            print("   total", tot, dict(c.most_common(14)))


if __name__ == "__main__":
    if sys.argv[1] == "ptxas":
        ptxas(sys.argv[2:])
    else:
        sass(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ".")
