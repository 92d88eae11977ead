"""Summarise an ncu report (raw metrics + stall breakdown + hot SASS)."""
import csv, json, subprocess, sys


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    d = dict(zip(r[0], r[2]))
    units = dict(zip(r[0], r[1]))
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if k in d:
            d[k + ".bytes"] = float(d[k].replace(",", "")) * SCALE.get(units.get(k, "byte"), 1)
    return d


def summary(rep):
    d = raw(rep)
    keys = ['Kernel Name', 'gpu__time_duration.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
            'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed.avg.per_cycle_active',
            'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
            'launch__grid_size', 'dram__bytes_read.sum.bytes', 'dram__bytes_write.sum.bytes',
            'smsp__thread_inst_executed_per_inst_executed.ratio',
            'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
            'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
            'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
            'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
            'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg.per_second']
    out = {k: d.get(k) for k in keys}
    f = lambda x: float((x or '0').replace(',', '') or 0)
    items = [(k, d[k]) for k in d if 'smsp__pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued')]
    tot = sum(f(x) for _, x in items) or 1
    out['stall_fractions'] = {k.replace('smsp__pcsamp_warps_issue_stalled_', ''): round(f(x) / tot, 3)
                              for k, x in sorted(items, key=lambda t: -f(t[1]))[:10]}
    return out


if __name__ == "__main__":
    print(json.dumps(summary(sys.argv[1]), indent=1))
