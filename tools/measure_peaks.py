"""Measure the SIMT pipe peaks of this B200 (FFMA, FFMA2, DFMA, MUFU rsqrt) and
write profiles/peaks_b200.json — the roofline denominators for the SF kernel,
which is bound by these pipes (not HBM, not tensor cores). Run on the GPU box:
    python tools/measure_peaks.py
"""
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2510_09204_b200", "libsfb_peaks.so")


def main():
    lib = ctypes.CDLL(SO)
    lib.sfb_peak.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
    lib.sfb_peak.restype = ctypes.c_double
    clocks = []
    stop = threading.Event()

    def sample():
        while not stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip().splitlines()[0]
                clocks.append([float(v) for v in out.split(",")])
            except Exception:
                pass
            time.sleep(0.2)

    th = threading.Thread(target=sample, daemon=True)
    th.start()
    res = {}
    for name, which, iters in (("fp32_ffma_tflops", 0, 200000), ("fp32_ffma2_tflops", 1, 100000),
                               ("fp64_dfma_tflops", 2, 50000), ("mufu_rsq_tops", 3, 50000)):
        v = max(lib.sfb_peak(which, bpsm, iters) for bpsm in (4, 8))
        res[name] = v / 1e12
        print(f"{name}: {v / 1e12:.2f}", flush=True)
    stop.set()
    th.join()
    sm = sorted(c[0] for c in clocks)
    res["sm_mhz_median"] = sm[len(sm) // 2] if sm else None
    res["sm_max_mhz"] = clocks[0][1] if clocks else None
    res["how"] = ("tools/measure_peaks.py: 148 SMs x {4,8} CTAs x 256 threads, 8 independent "
                  "chains per thread, best of 3 CUDA-event timings (csrc/peaks.cu)")
    out = os.path.join(ROOT, "profiles", "peaks_b200.json")
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    sys.exit(main())
