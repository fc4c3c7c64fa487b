"""profiles/<tag>_traffic.json: DRAM bytes (ncu dram__bytes_read.sum + dram__bytes_write.sum) per bench
step of each conv stage, from tools/gpu_traffic.sh's captures.  usage: python tools/traffic_json.py <tag>"""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1903_02440_b200 import snn  # noqa: E402  (host-only plan query, no GPU needed)


def launches(rep):
    txt = subprocess.run(["ncu", "-i", os.path.join(ROOT, "gpurun_out", rep), "--page", "raw", "--csv", "--print-units",
                          "base", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    h = r[0]
    return [(d["Kernel Name"], float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"]),
             float(d["gpu__time_duration.sum"])) for d in (dict(zip(h, x)) for x in r[2:])]


out = {}
k2 = launches("traffic_c2.ncu-rep")  # conv1 walk, conv2 sort + walk, conv3 (K9) prep limbs + prep_b + prep_a + tc
assert len(k2) == 7, [x[0][:30] for x in k2]
out["c2:conv1"] = k2[0][1]
out["c2:conv2"] = k2[1][1] + k2[2][1]
out["c2:conv3"] = sum(x[1] for x in k2[3:])
k5 = launches("traffic_c5.ncu-rep")  # 2 (sort, walk) chunk pairs of C5 conv1
chunks = snn.conv_fire_plan(64, 32, 256, 256, 2, 256, 5, 5, 32, 40.0)["chunks"]
out["c5:conv1"] = sum(x[1] for x in k5) / 2 * chunks
out["_note"] = ("DRAM bytes per bench step of the stage (all its launches), ncu --set full, "
                f"tools/gpu_traffic.sh; c5 scaled from 2 of {chunks} list chunks")
json.dump(out, open(os.path.join(ROOT, "profiles", f"{sys.argv[1]}_traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
