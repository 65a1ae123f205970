"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel."""
import collections, csv, sys

HARNESS = ("dmma_loop", "dfma_loop")


def is_harness(k):
    """sampler (the black-box operator, timed separately), the FP64 peak probe, torch kernels"""
    return k in HARNESS or k.startswith("matvec_") or k.startswith("at::")


def summarize(path):
    rows = list(csv.reader(open(path)))
    hdr_i = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hdr_i]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki]
        for pre in ("void ", "(anonymous namespace)::", "<unnamed>::", "rsrs::"):
            name = name.replace(pre, "")
        name = name.split("(")[0].split("<")[0].strip()
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
    tot = sum(v[1] for k, v in agg.items() if not is_harness(k))
    lines = []
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        sh = f"{100 * v[1] / tot:5.1f}%" if not is_harness(k) else "  (harness)"
        lines.append(f"{k:28s} n={v[0]:5d} total={v[1]:10.3f} ms  share_of_sweep={sh}")
    lines.append(f"sweep total (excl. harness/torch kernels) = {tot:.2f} ms")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
