"""Summarise a GPU measurement session (gpurun_out/) into profiles/: bench lines, per-kernel launch
shares (ncu gpu__time_duration list) and DRAM traffic of the captured kernels (ncu --set full).
usage: python tools/make_profile_summary.py <tag>      (writes profiles/<tag>_summary.md, _kernel_dram.json)"""
import collections, csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
tag = sys.argv[1]
out = [f"# GPU measurement summary `{tag}` (B200, sm_100a)\n"]

out.append("## Bench lines (`python bench.py --workload W`, default K/W)\n")
out.append("| workload | value | unit | ms/step | dominant | roofline frac | oracle (CPU) | e2e | SM MHz |")
out.append("|---|---|---|---|---|---|---|---|---|")
for w in ["c1", "c2", "c3", "c4", "c5"]:
    p = os.path.join(G, f"bench_{w}.json")
    if not os.path.exists(p):
        continue
    d = json.loads(open(p).read().strip().splitlines()[-1])
    rf = d.get("roofline") or {}
    out.append(f"| {w} | {d['value']:.1f} | {d['unit']} | {d['ms_per_step']:.3f} | {rf.get('kernel')} | "
               f"{rf.get('frac')} | {(d.get('cpu_baseline') or {}).get('value')} | {(d.get('e2e') or {}).get('value')} | "
               f"{(d.get('clocks') or {}).get('sm_mhz')} |")
    out.append(f"|  | stages (ms): {d.get('stages_ms')} |||||||| ")

out.append("\n## Kernel launch lists (ncu `gpu__time_duration.sum`, `--profile` run: cold, serialised; compare shares)\n")
for w in ["c1", "c2", "c3", "c4", "c5"]:
    p = os.path.join(G, f"launches_{w}.csv")
    if not os.path.exists(p):
        continue
    rows = list(csv.DictReader([l for l in open(p) if l.startswith('"')]))
    d = collections.OrderedDict()
    for r in rows:
        d.setdefault(r["Kernel Name"].split("(")[0], []).append(float(r["Metric Value"]) / 1e3)
    tot = sum(sum(v) for v in d.values())
    out.append(f"### {w}\n\n| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
    for k, v in d.items():
        out.append(f"| `{k}` | {len(v)} | {sum(v):.1f} | {sum(v)/len(v):.1f} | {sum(v)/tot:.3f} |")
    out.append("")

traffic = {}
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "launch__registers_per_thread"]
out.append("## ncu --set full captures (per launch)\n")
out.append("| report | kernel | us | DRAM read MB | DRAM write MB | issue active % | smem wavefronts/clk/SM | warps active % | regs |")
out.append("|---|---|---|---|---|---|---|---|---|")
for rep in sorted(f for f in os.listdir(G) if f.endswith(".ncu-rep")):
    txt = subprocess.run(["ncu", "-i", os.path.join(G, rep), "--page", "raw", "--csv", "--print-units", "base",
                          "--metrics", ",".join(M)], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    if len(r) < 3:
        continue
    h = r[0]
    for row in r[2:]:
        x = dict(zip(h, row))
        f = lambda k: float(x[k].replace(",", "")) if x.get(k) not in (None, "", "n/a") else float("nan")
        name = x["Kernel Name"].split("(")[0]
        us = f("gpu__time_duration.sum") / 1e3
        rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
        traffic.setdefault(rep.replace(".ncu-rep", "") + ":" + name, []).append(rd + wr)
        out.append(f"| {rep} | `{name}` | {us:.1f} | {rd/1e6:.1f} | {wr/1e6:.1f} | "
                   f"{f('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
                   f"{f('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum')/f('sm__cycles_elapsed.avg')/148:.2f} | "
                   f"{f('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | {x.get('launch__registers_per_thread')} |")
open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w").write("\n".join(out) + "\n")
json.dump({k: sum(v) / len(v) for k, v in traffic.items()}, open(os.path.join(ROOT, "profiles", f"{tag}_kernel_dram.json"), "w"),
          indent=1)
print("\n".join(out[:40]))
