"""Summarise ncu captures for profiles/: key metrics per kernel from
--set full reports and per-kernel shares from a launch-list CSV.
Usage: ncu_summary.py launches.csv rep1.ncu-rep [rep2 ...] > summary.md"""
import collections, csv, io, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active (% elapsed)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active (% SM-active)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe (% active)"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe (% active)"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue slots used (% active)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        k = r[ik].split("(")[0]
        tot[k] += float(r[iv].replace(",", "")) / 1e6
        cnt[k] += 1
    T = sum(tot.values())
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| `{k}` | {cnt[k]} | {v:.2f} | {100 * v / T:.1f} % |")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    for row in r[2:]:
        print(f"\n**`{row[h.index('Kernel Name')]}`** ({path.split('/')[-1]})\n")
        print("| metric | value |\n|---|---|")
        for k, name in KEYS:
            if k in h:
                i = h.index(k)
                print(f"| {name} (`{k}`) | {row[i]} {units[i]} |")


if __name__ == "__main__":
    launches(sys.argv[1])
    for p in sys.argv[2:]:
        full(p)
