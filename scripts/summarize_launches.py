"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``) into the
per-kernel table kept under profiles/: launches, total time, share, and the share of the
unit kernel within one bench step (the last launch of each hot-path kernel).

usage: python scripts/summarize_launches.py launches.csv "<command that produced it>" [note]
"""
import csv
import re
import sys
from collections import OrderedDict

HOT = ("lofp_table_off_kernel", "lofp_table_kernel", "lofp_tableA_kernel", "lofp_plan_kernel", "lofp_thr_kernel",
       "lofp_split_kernel", "lofp_scan_kernel", "lofp_units_kernel", "lofp_final_kernel", "lofp_generic_kernel",
       "lofp_contract_warp_kernel", "lofp_contract_kernel", "lofp_outputs_kernel")


def short(name: str) -> str:
    m = re.search(r"(lofp_\w+_kernel)(<[^>]*>)?", name)
    if m:
        tmpl = m.group(2) or ""
        return m.group(1) + tmpl.replace("(bool)", "").replace(" ", "")
    return name.replace("void ", "")[:60]


def main() -> None:
    path, cmd = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}[r["Metric Unit"]]
        rows.append((short(r["Kernel Name"]), float(r["Metric Value"].replace(",", "")) * scale))
    agg = OrderedDict()
    for k, ms in rows:
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + ms)
    tot = sum(t for _, t in agg.values())
    print(cmd)
    if note:
        print(note)
    print()
    print(f"{'kernel':60s} {'launches':>9s} {'total ms':>12s} {'share':>8s}")
    for k, (n, t) in agg.items():
        print(f"{k:60s} {n:9d} {t:12.3f} {100 * t / tot:7.2f}%")
    last = OrderedDict()
    for k, ms in rows:
        if any(k.split("<")[0] == h for h in HOT):
            last[k.split("<")[0]] = (k, ms)
    step = sum(ms for _, ms in last.values())
    print("\none step (last launch of each hot-path kernel: the timed, uncounted call):")
    for k, ms in last.values():
        print(f"  {k:50s} {ms:12.3f} ms {100 * ms / step:9.4f}% of the step")


if __name__ == "__main__":
    main()
