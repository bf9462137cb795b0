"""Opcode histogram of the hot loop of a kernel in a cubin/.o/.so: the instructions between
the first occurrence of START (an opcode regex, default LDS) and the backward branch that
closes the loop containing it.   python tools/loopstats.py <file> <kernel-regex> [START]"""
import collections, re, subprocess, sys

def kernels(path):
    txt = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    for fn in re.split(r"\n\s*Function : ", txt)[1:]:
        name = fn.split("\n")[0]
        dm = subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()
        ins = []
        for l in fn.split("\n"):
            m = re.search(r"/\*([0-9a-f]{4,5})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]+)([^;]*);", l)
            if m:
                ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
        yield dm, ins

def main():
    path, pat = sys.argv[1], sys.argv[2]
    start = sys.argv[3] if len(sys.argv) > 3 else "LDS"
    for dm, ins in kernels(path):
        if not re.search(pat, dm):
            continue
        first = next((i for i, x in enumerate(ins) if re.fullmatch(start, x[1])), None)
        if first is None:
            continue
        a0 = ins[first][0]
        # backward branch whose target is <= a0 and located after it: the enclosing loop
        best = None
        for i, (addr, op, rest) in enumerate(ins):
            if op == "BRA" and addr > a0:
                m = re.search(r"0x([0-9a-f]+)", rest)
                if m and int(m.group(1), 16) <= a0:
                    best = (int(m.group(1), 16), addr)
                    break
        if not best:
            print(dm[:100], "no loop found"); continue
        body = [op for addr, op, _ in ins if best[0] <= addr <= best[1] and op != "NOP"]
        c = collections.Counter(body)
        print(dm[:110])
        print("   loop body", len(body), "instructions:", dict(c.most_common(20)))

main()
