"""Measure the FP64 / FP32 / packed-FP32 FMA peaks (tools/fp_peak.cu) on the
GPU and write profiles/fp_peaks.json (run on the GPU box: nvcc is in the image)."""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def main():
    out_bin = os.path.join(ROOT, "build", "fp_peak")
    os.makedirs(os.path.dirname(out_bin), exist_ok=True)
    subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out_bin,
                    os.path.join(HERE, "fp_peak.cu")], check=True)
    res = json.loads(subprocess.run([out_bin], check=True, capture_output=True, text=True).stdout)
    res["how"] = ("tools/fp_peak.cu: 8 CTAs x 512 threads per SM, 8 independent FMA chains per "
                  "thread, best of 5 launches, CUDA events; flops = 2 per FMA lane")
    dst = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "fp_peaks.json")
    with open(dst, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
