"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel shares.

Usage: python tools/launch_shares.py gpurun_out/launches_c3.csv [title]
ncu's per-launch times are cold-cache and serialised, so compare SHARES of the step, not
absolute times, with the bench's own CUDA-event timings.
"""
import collections
import csv
import sys


def main() -> None:
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Value" in r)
    hdr = rows[hdr_i]
    ik, iu, iv = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    tot = collections.Counter()
    cnt = collections.Counter()
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
    for r in rows[hdr_i + 1:]:
        if len(r) <= iv:
            continue
        name = r[ik]
        if name.startswith("void "):
            name = name[5:]
        name = name.replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
        name = name.split("(")[0].split("<")[0].replace("rcp::", "")
        try:
            v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1e-6)
        except ValueError:
            continue
        tot[name] += v
        cnt[name] += 1
    # keep our own kernels (torch's setup kernels are outside the factorization)
    allt = sum(tot.values())
    print(f"total {allt:.2f} ms over {sum(cnt.values())} launches ({title}; ncu gpu__time_duration, "
          "--clock-control none; cold-cache, serialised: compare shares)")
    for name, v in tot.most_common():
        print(f"{100 * v / allt:5.1f}%  {v:9.2f} ms  {cnt[name]:5d}  {name}")


if __name__ == "__main__":
    main()
