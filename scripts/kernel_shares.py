"""Per-kernel share of a Ranker batch from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv`): the launches between
consecutive `ks_begin` markers (one fused step + K4 + its torch ops),
averaged over every complete batch after the first `skip` (warm-up).

    python scripts/kernel_shares.py gpurun_out/launches.csv [skip] > profiles/r2_cfg3_kernels.json
"""
import csv
import json
import sys


def main(path, skip=2):
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[h], rows[h + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    names = [r[ki] for r in data]
    marks = [i for i, n in enumerate(names) if "ks_begin" in n]
    segs = [data[a:b] for a, b in zip(marks[:-1], marks[1:])][skip:] or [data[marks[-2]:marks[-1]]]
    # one batch = one K4 launch (bench.py also times K4 alone between batches)
    segs = [g for g in segs if sum("k_pool" in r[ki] for r in g) == 1] or segs
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = {}
    for seg in segs:
        for r in seg:
            nm = r[ki].split("(")[0].replace("void ", "")
            nm = nm.split("<")[0] if nm.startswith("fx::") or nm.startswith("stp::") else nm[:60]
            agg[nm] = agg.get(nm, 0.0) + float(r[vi].replace(",", "")) * scale[r[ui]] / len(segs)
    tot = sum(agg.values())
    out = {"source": path, "batches_averaged": len(segs),
           "launches_per_batch": round(sum(len(g) for g in segs) / len(segs), 1),
           "serialized_us_per_batch": round(tot, 1),
           "note": "ncu launch list (cold-cache, serialised; shares, not absolute times)",
           "kernels": [{"kernel": k, "us": round(v, 1), "share": round(v / tot, 4)}
                       for k, v in sorted(agg.items(), key=lambda kv: -kv[1])]}
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 2)
