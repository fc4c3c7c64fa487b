"""One step of every workload at a shrunken batch, for compute-sanitizer (tools/gpu_sanitize.sh).

python tools/sanitize_run.py c1|c2|c3|c4|c5 -- builds the bench step object of that workload at a
small batch (C2 16 images, C3 48 images through the persistent kernel, C4 6 images through the
theta = +inf R-STDP sequence, C5 1 image), runs one step plus a second replay, synchronises and reads
the device error word.  Every kernel of the step runs under the sanitizer; no oracle is involved.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1903_02440_b200 import snn  # noqa: E402

BATCH = {"c1": 1, "c2": 16, "c3": 48, "c4": 6, "c5": 1}


def main():
    name = sys.argv[1]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    snn.lib()
    step = bench.WORKLOADS[name](torch, dev, batch=BATCH[name])
    for _ in range(2):
        step.run()
    torch.cuda.synchronize()
    snn.sync_status()
    print(f"{name}: ok (batch {BATCH[name]})", flush=True)


if __name__ == "__main__":
    main()
