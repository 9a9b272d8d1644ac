"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel.

    python tools/launch_summary.py gpurun_out/launches_c2.csv [--per lt::k_pencil]

Per-solve averages are normalised by the number of launches of the `--per` kernel
(default: the pencil / sygvd kernel, launched once per solve). ncu times are
cold-cache and serialised: compare shares, not absolutes.
"""
import argparse
import collections
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--per", default=None)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    ours = {k: v for k, v in tot.items() if k.startswith("lt::") or "cusolver" in k.lower() or "syevd" in k.lower()}
    per_key = a.per
    if per_key is None:
        cands = [k for k in cnt if "k_pencil" in k] or [k for k in cnt if "k_triv_reduce_w" in k or "k_fill" in k]
        per_key = cands[0] if cands else max(cnt, key=cnt.get)
    solves = max(1, cnt[per_key])
    s = sum(tot.values())
    print(f"{a.csv}: {solves} solves (normalised by {per_key}); all kernels {s / solves / 1e3:.1f} us/solve")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:25]:
        print(f"  {k:55s} {v / solves / 1e3:9.1f} us/solve  {cnt[k] / solves:5.1f} launches  share {v / s:.3f}")


if __name__ == "__main__":
    main()
