"""Per-launch gpu__time_duration from an ncu --csv log: `python tools/ncu_times.py log.csv`."""
import csv
import io
import re
import sys


def main(path):
    text = open(path).read()
    text = text[text.find('"ID"'):]
    for r in csv.DictReader(io.StringIO(text)):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("(anonymous namespace)::", "")
        print(f'{r["ID"]:>4} {name[:48]:<48} {float(r["Metric Value"]) / 1e3:9.2f} us')


if __name__ == "__main__":
    main(sys.argv[1])
