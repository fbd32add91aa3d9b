"""Summarise `nvcc -Xptxas -v` logs: kernel -> registers / spills / smem."""
import glob
import re
import subprocess
import sys

def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.splitlines()

def main(pattern):
    rows = []
    for f in sorted(glob.glob(pattern)):
        cur = None
        for line in open(f):
            m = re.search(r"Compiling entry function '(\S+)'", line)
            if m:
                cur = [m.group(1), "", "", ""]
                rows.append(cur)
                continue
            if cur is None:
                continue
            m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
            if m:
                cur[2] = f"spill {m.group(1)}/{m.group(2)}"
            m = re.search(r"Used (\d+) registers.*?(\d+) bytes smem", line)
            if m:
                cur[1] = f"regs {m.group(1)}"
                cur[3] = f"smem {m.group(2)}"
            elif re.search(r"Used (\d+) registers", line):
                cur[1] = "regs " + re.search(r"Used (\d+) registers", line).group(1)
    names = demangle([r[0] for r in rows])
    for n, r in zip(names, rows):
        n = re.sub(r"\(.*", "", n).replace("dw::", "").replace("(anonymous namespace)::", "")
        print(f"{n:60s} {r[1]:10s} {r[2]:14s} {r[3]}")

if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "paper_2401_05345_b200/csrc/build/*.ptxas.txt")
