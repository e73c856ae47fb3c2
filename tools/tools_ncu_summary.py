"""tools_ncu_summary.py REPORT.ncu-rep -- per-kernel summary of an `ncu --set full` report
(speed-of-light, occupancy, stall reasons, DRAM traffic), read with `ncu -i` in this container."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def page(name):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


det = page("details")
hdr = det[0]
ix = {h: i for i, h in enumerate(hdr)}
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Compute (SM) Throughput", "Executed Ipc Active", "Registers Per Thread",
        "Theoretical Occupancy", "Achieved Occupancy", "Dynamic Shared Memory Per Block"]
kern = {}
for r in det[1:]:
    k = (r[ix["ID"]], r[ix["Kernel Name"]])
    if r[ix["Metric Name"]] in want:
        kern.setdefault(k, []).append(f"{r[ix['Metric Name']]} {r[ix['Metric Value']]} {r[ix['Metric Unit']]}")
raw = page("raw")
rh, units = raw[0], raw[1]


def f(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for (kid, name), lines in kern.items():
    print(f"## [{kid}] {name[:110]}")
    for l in lines:
        print("   " + l)
    row = next((r for r in raw[2:] if r[rh.index("ID")] == kid), None)
    if row is None:
        continue
    d = dict(zip(rh, row))
    st = sorted([(f(v), h) for h, v in d.items()
                 if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued") and f(v)], reverse=True)[:6]
    print("   stalls: " + ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')}={s:.0f}" for s, h in st))
    rd = f(d["dram__bytes_read.sum"]) * scale.get(units[rh.index("dram__bytes_read.sum")], 1)
    wr = f(d["dram__bytes_write.sum"]) * scale.get(units[rh.index("dram__bytes_write.sum")], 1)
    print(f"   dram read {rd / 1e9:.4f} GB, write {wr / 1e9:.4f} GB, traffic {(rd + wr) / 1e9:.4f} GB")
    for h in ["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
              # the L1 return path (64 B per wavefront and cycle per SM): the gathers' bound
              "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
              "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg",
              "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum", "sm__cycles_elapsed.max"]:
        if h in d:
            print(f"   {h} {d[h]}")
