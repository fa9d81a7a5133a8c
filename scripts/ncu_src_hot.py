"""Aggregate an `ncu --page source --csv --print-source cuda,sass` export by source line.

Prints the hottest source lines (warp-stall samples) with their top stall reasons.
  ncu -i rep --page source --csv --print-source cuda,sass --kernel-name regex:K \
      --launch-skip S --launch-count 1 > src.csv; python scripts/ncu_src_hot.py src.csv [N]
"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = list(csv.reader(open(path)))
    fname, hdr, line, src = None, None, None, None
    agg = defaultdict(lambda: defaultdict(float))
    text = {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        if r[0]:
            line, src = int(r[0]), r[1]
            text[(fname, line)] = src.strip()
            continue
        if r[2] in ("-", "..."):
            continue
        key = (fname, line)
        for i, h in enumerate(hdr):
            if i < 4:
                continue
            if h in ("Warp Stall Sampling (All Samples)", "Instructions Executed") or (h.startswith("stall_") and "Not Issued" not in h):
                try:
                    agg[key][h] += float(r[i])
                except ValueError:
                    pass
    tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values())
    itot = sum(v["Instructions Executed"] for v in agg.values())
    print(f"total warp instructions executed {itot:.0f}")
    if len(sys.argv) > 3:  # per line-range totals: file:lo-hi,... (instructions, stall samples)
        for spec in sys.argv[3].split(","):
            f, rng = spec.split(":")
            lo, hi = map(int, rng.split("-"))
            ins = sum(v["Instructions Executed"] for (ff, ln), v in agg.items() if ff == f and lo <= ln <= hi)
            smp = sum(v["Warp Stall Sampling (All Samples)"] for (ff, ln), v in agg.items() if ff == f and lo <= ln <= hi)
            print(f"  {spec:30s} instr {100 * ins / max(itot, 1):5.1f}%  samples {100 * smp / max(tot, 1):5.1f}%")
    hot = sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:top]
    print("-- hottest by stall samples (i = share of executed instructions)")
    for (f, ln), v in hot:
        s = v["Warp Stall Sampling (All Samples)"]
        reasons = sorted(((k[6:], x) for k, x in v.items() if k.startswith("stall_")), key=lambda t: -t[1])[:3]
        rs = " ".join(f"{k}:{100 * x / max(s, 1):.0f}%" for k, x in reasons if x > 0)
        ins = v["Instructions Executed"]
        print(f"{100 * s / tot:5.1f}% i{100 * ins / max(itot, 1):5.1f}% {f}:{ln:<5} {rs:40s} {text.get((f, ln), '')[:70]}")


if __name__ == "__main__":
    main()
