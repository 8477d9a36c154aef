"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-launch time and
share of the listed total (cold-cache, serialised: compare shares, not absolutes)."""
import csv
import sys


def main(path, last=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    recs = [dict(zip(h, r)) for r in rows[1:] if dict(zip(h, r)).get("Metric Name") ==
            "gpu__time_duration.sum"]
    if last:
        recs = recs[-int(last):]
    unit = recs[0]["Metric Unit"] if recs else ""
    tot = sum(float(r["Metric Value"].replace(",", "")) for r in recs)
    for r in recs:
        v = float(r["Metric Value"].replace(",", ""))
        print(f"{v:12.3f} {unit:5s} {100 * v / tot:5.1f}%  {r['Kernel Name'][:80]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
