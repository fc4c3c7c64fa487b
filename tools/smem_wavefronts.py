"""profiles/<tag>_smem_wavefronts.json: shared-memory wavefronts of the finite-threshold walk kernels (ncu --set
full captures of tools/gpu_traffic.sh: gpurun_out/traffic_c2.ncu-rep, traffic_c5.ncu-rep; metric
l1tex__data_pipe_lsu_wavefronts_mem_shared.sum) against the useful wavefronts = necessary events x 4 B / 128 B
(the roofline's algorithmic work, from the committed bench lines profiles/<tag>_bench_c2/c5.json).
usage: python tools/smem_wavefronts.py <tag>"""
import csv, io, json, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1903_02440_b200 import snn  # noqa: E402  (host-only plan query)

tag = sys.argv[1]
M = ["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg", "gpu__time_duration.sum"]


def launches(rep):
    txt = subprocess.run(["ncu", "-i", os.path.join(ROOT, "gpurun_out", rep), "--page", "raw", "--csv", "--print-units",
                          "base", "--metrics", ",".join(M)], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    h = r[0]
    return [dict(zip(h, x)) for x in r[2:]]


def necessary(w):
    d = json.load(open(os.path.join(ROOT, "profiles", f"{tag}_bench_{w}.json")))
    rf = d["roofline"] if w == "c5" else None
    work = (rf or d["roofline"])["work"]
    return int(re.match(r"(\d+) necessary events", work).group(1))


f = lambda x, k: float(x[k].replace(",", ""))
out = {"_note": __doc__.split("usage")[0].strip()}
k2 = [x for x in launches("traffic_c2.ncu-rep") if "conv_walk_kernel" in x["Kernel Name"]]
walk2 = k2[1]  # conv1's row-tile walk, then conv2's presorted walk
wf, useful = f(walk2, M[0]), necessary("c2") * 4 / 128
out["c2_conv2_walk"] = {"wavefronts": int(wf), "useful": int(useful), "useful_frac": round(useful / wf, 3),
                        "crossbar_busy": round(wf / f(walk2, M[1]) / 148, 3), "us": round(f(walk2, M[2]) / 1e3, 1)}
k5 = [x for x in launches("traffic_c5.ncu-rep") if "conv_walk_kernel" in x["Kernel Name"]]
chunks = snn.conv_fire_plan(64, 32, 256, 256, 2, 256, 5, 5, 32, 40.0)["chunks"]
full, last = f(k5[0], M[0]), f(k5[1], M[0])  # a full list chunk and the partial last one
wf5, useful5 = full * (chunks - 1) + last, necessary("c5") * 4 / 128
out["c5_conv1_walk"] = {"wavefronts_per_step": int(wf5), "useful_per_step": int(useful5),
                        "useful_frac": round(useful5 / wf5, 3),
                        "wavefronts_per_clk_per_sm": round(full / f(k5[0], M[1]) / 148, 3),
                        "us_per_full_chunk": round(f(k5[0], M[2]) / 1e3, 1), "chunks": chunks}
json.dump(out, open(os.path.join(ROOT, "profiles", f"{tag}_smem_wavefronts.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
