"""Summarise an ncu report: key raw metrics + stall reasons + hottest SASS (debug helper).
   python tools/ncu_summary.py gpurun_out/prof_output.ncu-rep [nsass]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
nsass = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum"]
for k in keys:
    if k in hdr:
        i = hdr.index(k)
        print("%-66s %s %s" % (k, vals[i], units[i]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[ix[k]])
    except Exception: return 0.0
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
print("stall samples", tot)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {s: sum(f(r, s) for r in data) for s in stalls}
print("  " + "  ".join("%s %.1f%%" % (s[6:], 100 * v / tot) for s, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:nsass]:
    print("%6.2f%% n=%9d  %s" % (100 * f(r, "Warp Stall Sampling (All Samples)") / tot,
                                 f(r, "Instructions Executed"), r[ix["Source"]][:100]))
