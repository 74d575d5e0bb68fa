"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of
`bench.py --steps 1 --warmup 1`: splits the launches into training steps at the
optimizer's multi-tensor-apply kernels and prints the per-kernel totals of step N
(default: the second = the timed step).  Times are ncu's serialized cold-cache
durations -- compare shares, not absolutes.

  python tools/launch_summary.py gpurun_out/launches.csv [step_index]
"""
import collections
import csv
import sys

UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
        "second": 1e3, "s": 1e3}


def main(path, step=1):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    ik, iv, iu, im = (h.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit",
                                            "Metric Name"))
    launches = [(r[ik], float(r[iv].replace(",", "")) * UNIT[r[iu]]) for r in rows[1:]
                if r[im] == "gpu__time_duration.sum"]
    steps, cur, in_opt = [], [], False
    for name, ms in launches:
        opt = ("FusedOptimizerTensorListMetadata" in name or "FusedAdamW" in name or
               "adamw_bf16_kernel" in name)
        if in_opt and not opt:
            steps.append(cur)
            cur = []
        in_opt = opt
        cur.append((name, ms))
    steps.append(cur)
    sel = steps[step]
    tot = sum(ms for _, ms in sel)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, ms in sel:
        agg[name][0] += 1
        agg[name][1] += ms
    print(f"{len(steps)} steps found; step {step}: {len(sel)} launches, {tot:.1f} ms summed "
          f"kernel time (ncu, serialized, cold-cache)")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        if v / tot < 0.001:
            continue
        print(f"{v:9.2f} ms {v / tot * 100:5.1f}% x{c:4d} {k[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
