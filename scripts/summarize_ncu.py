"""Summarise ncu artefacts into profiles/: per-kernel launch list shares (from the
gpu__time_duration launch list) and key metrics of the full capture."""
import csv, collections, json, subprocess, sys

def launch_list(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]; ki, vi = h.index('Kernel Name'), h.index('Metric Value')
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        name = r[ki].split('(')[0].replace('void ', '').replace('vinf::', '').replace('<unnamed>::', '')
        agg.setdefault(name, []).append(float(r[vi].replace(',', '')) / 1000.0)
    return agg

def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines())); h = rows[0]
    want = {"time_us": "gpu__time_duration.sum", "dram_read_MB": "dram__bytes_read.sum",
            "dram_write_MB": "dram__bytes_write.sum",
            "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "lts_hit_pct": "lts__t_sector_hit_rate.pct",
            "issue_active_pct": "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
            "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
            "regs": "launch__registers_per_thread", "smem_KB": "launch__shared_mem_per_block_dynamic"}
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split('(')[0][:60]}
        for k, m in want.items():
            if m in h:
                try: d[k] = float(r[h.index(m)])
                except ValueError: d[k] = r[h.index(m)]
        res.append(d)
    return res

if __name__ == "__main__":
    ll = launch_list(sys.argv[1])
    print("# launch list (ncu gpu__time_duration.sum, cold-cache, serialised)")
    tot = sum(sum(v) for k, v in ll.items() if 'fill_seeded' not in k and 'split_kernel' not in k)
    for k, v in ll.items():
        print(f"{len(v):4d} launches  avg {sum(v)/len(v):9.1f} us  share {sum(v)/tot:6.3f}  {k}")
    if len(sys.argv) > 2:
        print("\n# full capture (--set full), one launch each")
        for d in full(sys.argv[2]):
            print(json.dumps(d))
