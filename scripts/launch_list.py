"""Turn an `ncu --metrics gpu__time_duration.sum --csv` launch list into a markdown table of
one bench step (from the first input pass / first conv to the following argmax, or to the
next step when the last layer writes the labels itself)."""
import csv
import sys


def main(path, out, title):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr = rows[0]
    ik, im, iv, iid = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    ks = [(int(r[iid]), r[ik], float(r[iv].replace(",", ""))) for r in rows[1:] if r[im] == "gpu__time_duration.sum"]
    # the step: from the first input pass (or first conv) to the next argmax_kernel (inclusive)
    starts = [i for i, k in enumerate(ks) if "input_rows" in k[1] or "check_finite" in k[1]]
    if not starts:  # the first conv checks its input itself (fused input pass): it opens the step
        starts = [i for i, k in enumerate(ks) if "first_conv" in k[1]]
    s0 = starts[0]
    # ... to the step's argmax, or (labels fused into the last layer) up to the next step's start
    e0 = next((i for i in range(s0, len(ks)) if "argmax" in ks[i][1]), None)
    if e0 is None:
        e0 = next((i - 1 for i in range(s0 + 1, len(ks)) if ks[i][1] == ks[s0][1]), len(ks) - 1)
    step = ks[s0:e0 + 1]
    tot = sum(k[2] for k in step) / 1e3
    with open(out, "w") as f:
        f.write(f"# {title}\n\n`ncu --metrics gpu__time_duration.sum --clock-control none` of the bench command; launches "
                f"{step[0][0]}-{step[-1][0]} are one step. Cold-cache and serialized: compare shares, not absolutes "
                f"(sum {tot:.1f} us).\n\n| launch | kernel | time (us) | share |\n|---|---|---|---|\n")
        for i, name, ns in step:
            f.write(f"| {i} | `{name[:90]}` | {ns / 1e3:.1f} | {100 * ns / 1e3 / tot:.1f}% |\n")
    print(out, len(step), "launches", f"{tot:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "ncu launch list")
