"""Top SASS lines of one kernel in an ncu report by stall samples / executed
instructions: `python tools/ncu_hotspots.py rep.ncu-rep regex:k_name [N]`."""
import csv
import io
import subprocess
import sys


def main(rep, kernel, n=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kernel,
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = [r for r in csv.DictReader(io.StringIO("\n".join(lines[start:])))
            if r["Address"] != "Address"]  # one header per kernel instance
    seen, uniq = set(), []
    for r in rows:  # first instance only
        if r["Address"] in seen:
            break
        seen.add(r["Address"])
        uniq.append(r)
    rows = uniq
    tot_s = sum(float(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    tot_i = sum(float(r["Instructions Executed"] or 0) for r in rows)
    print(f"samples {tot_s:.0f}  warp-inst {tot_i:.0f}  sass lines {len(rows)}")
    rows.sort(key=lambda r: -float(r["Warp Stall Sampling (All Samples)"] or 0))
    for r in rows[:int(n)]:
        print(f'{float(r["Warp Stall Sampling (All Samples)"] or 0):7.0f} '
              f'{float(r["Instructions Executed"] or 0):10.0f}  {r["Address"][-5:]}  {r["Source"].strip()[:70]}')


if __name__ == "__main__":
    main(*sys.argv[1:])
