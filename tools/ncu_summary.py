"""Summarise an ncu --set full report (one kernel launch) as markdown for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--algo-bytes B] > profiles/x.md

Reads the raw page (DRAM bytes, duration, pipe utilisation, warp-stall sampling)
and, if present, the SASS source page (instruction mix, instructions per element).
"""
import argparse
import collections
import csv
import io
import subprocess


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--algo-bytes", type=float, default=None, help="algorithmic bytes per launch")
    ap.add_argument("--elements", type=float, default=None, help="logits elements per launch")
    ap.add_argument("--title", default=None)
    a = ap.parse_args()
    raw = ncu_csv(a.rep, "--page", "raw")
    hdr, units, vals = raw[0], raw[1], raw[2]
    d = {hdr[i]: (vals[i], units[i]) for i in range(len(hdr))}
    name = d.get("Kernel Name", ("?", ""))[0]
    print(f"## {a.title or name}\n")
    print(f"kernel: `{name}`  grid {d.get('launch__grid_size', ('?',))[0]} x block "
          f"{d.get('launch__block_size', ('?',))[0]}, regs/thread "
          f"{d.get('launch__registers_per_thread', ('?',))[0]}\n")
    keys = [
        ("gpu__time_duration.sum", "duration"),
        ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
        ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
        ("smsp__inst_executed.sum", "warp instructions executed"),
        ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ]
    print("| metric | value |\n|---|---|")
    for k, label in keys:
        if k in d:
            print(f"| {label} (`{k}`) | {d[k][0]} {d[k][1]} |")
    traffic = None
    try:
        def gb(k):
            v, u = d[k]
            v = float(v.replace(",", ""))
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]
        traffic = gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")
        print(f"| DRAM traffic (read+write) | {traffic:.4g} B |")
        if a.algo_bytes:
            print(f"| algorithmic bytes | {a.algo_bytes:.4g} B (traffic / algorithmic = "
                  f"{traffic / a.algo_bytes:.3f}) |")
    except Exception:
        pass
    st = [(k, float(v.replace(",", ""))) for k, (v, u) in d.items()
          if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")]
    tot = sum(x for _, x in st) or 1.0
    print("\nwarp-state samples (top):\n\n| reason | share |\n|---|---|")
    for k, x in sorted(st, key=lambda t: -t[1])[:8]:
        print(f"| {k.replace('smsp__pcsamp_warps_issue_stalled_', '')} | {100 * x / tot:.1f}% |")
    src = ncu_csv(a.rep, "--page", "source", "--print-source=sass")
    if len(src) > 3 and "Instructions Executed" in src[1]:
        ie = src[1].index("Instructions Executed")
        rows = src[2:]
        ops = collections.Counter()
        total = 0
        for r in rows:
            if r and r[0] == "Kernel Name":  # next launch in the report: first one only
                break
            if len(r) <= ie or not r[ie].isdigit():
                continue
            t = r[1].strip().split()
            if not t:
                continue
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            n = int(r[ie])
            ops[op] += n
            total += n
        print(f"\nSASS mix ({total} warp instructions"
              + (f"; {total * 32 / a.elements:.2f} thread instructions per logit" if a.elements else "")
              + "):\n\n| op | share |\n|---|---|")
        for op, n in ops.most_common(12):
            print(f"| {op} | {100 * n / total:.1f}% |")
    print()


if __name__ == "__main__":
    main()
