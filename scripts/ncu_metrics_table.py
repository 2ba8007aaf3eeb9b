"""Tabulate an ncu --csv metrics log: one row per launch, one column per metric."""
import csv, sys
from collections import OrderedDict

def load(path):
    rows = OrderedDict()
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        key = int(r["ID"])
        d = rows.setdefault(key, {"kernel": r["Kernel Name"].split("(")[0][-40:]})
        try:
            d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            d[r["Metric Name"]] = r["Metric Value"]
    return rows

if __name__ == "__main__":
    rows = load(sys.argv[1])
    cols = [c for c in next(iter(rows.values())).keys() if c != "kernel"]
    print("id  " + "  ".join(c.split("__")[-1][:22].rjust(22) for c in cols))
    for k, d in rows.items():
        print(f"{k:3d} " + "  ".join(f"{d.get(c, 0):22.4g}" if isinstance(d.get(c, 0), float) else str(d.get(c)).rjust(22) for c in cols))
