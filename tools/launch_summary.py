"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.
    python tools/launch_summary.py gpurun_out/launches.csv NFACT > profiles/ncu_launches_..._summary.txt
NFACT = number of factorizations in the run (the per-factorization numbers are totals / NFACT).
libhf kernels (namespace hf::) first, then the library kernels (cuBLASLt) apart."""
import csv
import re
import sys
from collections import defaultdict


def main(path, nfact):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ik, iv, ig = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
    tot = defaultdict(lambda: [0, 0.0])
    lib = defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = r[ik]
        if not re.search(r"(hf::|p32::|p64::)", name):
            # library kernels (cuBLASLt's int8 / bf16 GEMMs of ozaki.cu and k_trsm_blk.cu,
            # torch's copies): listed apart
            short = re.sub(r"^void ", "", name).split("(")[0][:48]
            lib[short][0] += 1
            lib[short][1] += float(r[iv].replace(",", ""))
            continue
        short = re.sub(r"^void ", "", name)
        short = re.sub(r"(hf::)?(p32::|p64::)?(\(anonymous namespace\)|<unnamed>)::", "", short)
        short = short.split("(")[0]
        tot[short][0] += 1
        tot[short][1] += float(r[iv].replace(",", ""))
    allns = sum(v[1] for v in tot.values())
    print(f"{'kernel':34s} {'launches':>9s} {'ms':>9s} {'share':>7s}   (per factorization)")
    for k, (n, ns) in sorted(tot.items(), key=lambda x: -x[1][1]):
        print(f"{k:34s} {n / nfact:9.1f} {ns / nfact / 1e6:9.2f} {100 * ns / allns:6.1f}%")
    print(f"{'total':34s} {sum(v[0] for v in tot.values()) / nfact:9.1f} {allns / nfact / 1e6:9.2f}")
    if lib:
        libns = sum(v[1] for v in lib.values())
        print(f"\nlibrary kernels (not libhf's; per factorization): {sum(v[0] for v in lib.values()) / nfact:.1f} "
              f"launches, {libns / nfact / 1e6:.2f} ms")
        for k, (n, ns) in sorted(lib.items(), key=lambda x: -x[1][1])[:15]:
            print(f"  {k:48s} {n / nfact:9.1f} {ns / nfact / 1e6:9.2f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
