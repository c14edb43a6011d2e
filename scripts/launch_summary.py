"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a
per-kernel share table (markdown).  ncu's per-launch times are cold-cache and
serialised: compare SHARES, not absolute times."""
import collections, csv, sys

def main(path, out, title):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        v = v / 1000 if r[ui] == "ns" else (v * 1000 if r[ui] == "ms" else v)
        name = r[ki].split("(")[0].replace("void ", "").strip()[:70]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    with open(out, "w") as f:
        f.write(f"# {title}\n\nsource: `{path}` ({sum(cnt.values())} launches, {T/1e3:.1f} ms total, "
                "ncu cold-cache serialised times — shares only)\n\n| share | total us | launches | kernel |\n|---:|---:|---:|---|\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            f.write(f"| {v / T * 100:.2f}% | {v:.1f} | {cnt[k]} | `{k}` |\n")
    print(open(out).read())

if __name__ == "__main__":
    main(*sys.argv[1:])
