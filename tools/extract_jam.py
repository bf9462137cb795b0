"""One-time transcription of the JAM-scaled matrices T(16) and T(32) printed in PAPER.md
(§6.2 "Video Coding") into oracle/data/t16.txt and oracle/data/t32.txt.

Run on the dev box (the paper text is not on the GPU box):  python tools/extract_jam.py
The files are committed; tests/test_oracle_jam.py pins them to the JAM recursion (Eq. 7,
P:L2617-2660) applied to T1, to the printed D(16)/D(32) and to Table 8.
"""
import re
import sys

PAPER = "/root/reference/PAPER.md"


def matrices(lines):
    out, cur = [], None
    for ln in lines:
        if "begin{smallmatrix}" in ln:
            cur = []
            continue
        if "end{smallmatrix}" in ln:
            out.append(cur)
            cur = None
            continue
        if cur is not None and "&" in ln:
            row = ln.replace("\\phantom{-}", "").replace("\\\\", "").strip()
            try:
                cur.append([int(v) for v in row.split("&")])
            except ValueError:  # the 2x2 identities of D(16), D(32) are written on one line
                cur.append([])
    return out


def main():
    lines = open(PAPER).read().split("\n")
    start = next(i for i, l in enumerate(lines) if "mathbf{T}_{(16)}" in l)
    ms = [m for m in matrices(lines[start:start + 120]) if len(m) in (16, 32)]
    t16 = next(m for m in ms if len(m) == 16)
    t32 = next(m for m in ms if len(m) == 32)
    for name, m, lo in (("t16", t16, start + 1), ("t32", t32, start + 1)):
        assert all(len(r) == len(m) for r in m), name
        with open(f"oracle/data/{name}.txt", "w") as f:
            f.write(f"# {name.upper()} = the JAM-scaled {len(m)}-point T1 printed in PAPER.md §6.2 "
                    f"(P:L2669-2739), transcribed by tools/extract_jam.py\n")
            for r in m:
                f.write(" ".join(f"{v:2d}" for v in r) + "\n")
    print("wrote", len(t16), len(t32))


if __name__ == "__main__":
    sys.exit(main())
