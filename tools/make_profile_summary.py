"""Turn the ncu artefacts of one round (gpurun_out/<tag>_*) into committed text under profiles/."""
import collections, csv, io, json, os, subprocess, sys

tag = sys.argv[1]
src = "gpurun_out"
out = [f"# {tag}: ncu evidence (tools/r02_evidence.sh {tag} / tools/ncu_round.sh {tag})\n"]
rows = [r for r in csv.reader(open(f"{src}/{tag}_launches_c4_xyz_16_2.csv")) if len(r) > 5 and r[0].isdigit()]
agg = collections.OrderedDict()
for r in rows:
    a = agg.setdefault(r[4].split("(")[0], [0, 0.0])
    a[0] += 1
    a[1] += float(r[-1].replace(",", ""))
tot = sum(v[1] for v in agg.values())
out.append("\n## launch list, xyz_chain(16,2) v3, warm-up + 1 step (ncu --metrics gpu__time_duration.sum --clock-control none)\n")
out.append(f"{'kernel':44s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}\n")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"{k[:44]:44s} {v[0]:8d} {v[1] / 1e6:10.3f} {v[1] / tot:7.1%}\n")
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]
traffic = {}
for name in sorted(os.listdir(src)):
    if not (name.startswith(tag + "_") and name.endswith(".ncu-rep")):
        continue
    txt = subprocess.run(["ncu", "-i", f"{src}/{name}", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(txt)))
    if len(rr) < 3:
        continue
    hdr, units, r = rr[0], rr[1], rr[2]
    v1 = name.startswith(tag + "_v1_")
    wl = "xyz_chain(14,2) v1" if v1 else "config 5 (32 qubits, 5000 gates) v3, the whole circuit" if "k_small_circuit" in name else "xyz_chain(16,2) v3"
    out.append(f"\n## {name[len(tag) + 1:-8]} ({wl}, ncu --set full, first captured launch): {r[hdr.index('Kernel Name')][:70]}\n")
    for w in want:
        if w in hdr:
            out.append(f"{w:78s} {r[hdr.index(w)]:>16s} {units[hdr.index(w)]}\n")
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
            try:
                stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    out.append("stalls (warps per issue): " + ", ".join(f"{n}={v:.2f}" for v, n in sorted(stalls, reverse=True)[:6]) + "\n")
    def gb(col):
        v, u = float(r[hdr.index(col)]), units[hdr.index(col)]
        return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[u]
    if "k_onesweep" in name and not v1:
        traffic["sort_pass"] = gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")
    if "k_bucket_emit" in name and not v1:
        traffic["bucket_emit"] = gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")
open(f"profiles/{tag}_summary.txt", "w").writelines(out)
if traffic:
    old = json.load(open("profiles/traffic.json")) if os.path.exists("profiles/traffic.json") else {}
    old.update(traffic)
    json.dump(old, open("profiles/traffic.json", "w"))
print("".join(out))
