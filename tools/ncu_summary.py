"""One-screen summary of ncu --set full reports (duration, DRAM bytes,
instructions, issue / SM throughput, occupancy, registers, local-memory,
L2 atomic / write sectors, bulk-copy instructions, top stall reasons).
Usage: python tools/ncu_summary.py name=report.ncu-rep ..."""
import csv, re, subprocess, sys

WANT = [
    ("duration", "gpu__time_duration.sum"),
    ("DRAM read", "dram__bytes_read.sum"),
    ("DRAM write", "dram__bytes_write.sum"),
    ("warp instructions", "smsp__inst_executed.sum"),
    ("SM throughput %", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("issue active %", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("IPC", "sm__inst_executed.avg.per_cycle_active"),
    ("warps active / SM", "sm__warps_active.avg.per_cycle_active"),
    ("registers/thread", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("local-memory load sectors", "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum"),
    ("L2 atomic sectors", "lts__t_sectors_srcunit_tex_op_atom.sum"),
    ("L2 atomic sectors % of peak", "lts__t_sectors_srcunit_tex_op_atom.sum.pct_of_peak_sustained_elapsed"),
    ("L2 reduction sectors", "lts__t_sectors_srcunit_tex_op_red.sum"),
    ("L2 write sectors", "lts__t_sectors_srcunit_tex_op_write.sum"),
    ("L2 write sectors % of peak", "lts__t_sectors_srcunit_tex_op_write.sum.pct_of_peak_sustained_elapsed"),
    ("L2 throughput %", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed"),
    ("DRAM throughput %", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("shared-memory wavefronts %", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    ("L2 hit rate %", "lts__t_sector_hit_rate.pct"),
]


def report(name, rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    print(f"### {name}  ({d.get('Kernel Name', '')[:90]})")
    for label, key in WANT:
        if key in d:
            print(f"  {label:28s} {d[key]:>22s} {u.get(key, '')}")
    stalls = []
    for k, val in d.items():
        m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$", k)
        if m and val:
            try:
                stalls.append((float(val.replace(",", "")), m.group(1)))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    print("  top stalls per issue:", ", ".join(f"{n} {x:.2f}" for x, n in stalls[:5]))


for arg in sys.argv[1:]:
    n, r = arg.split("=", 1)
    report(n, r)
