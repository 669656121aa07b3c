"""Measure FP32 (FFMA, FFMA2) and FP64 (DFMA, DMMA) peak throughput on this
GPU and the SM clock during the run; print one JSON line.

    python tools/peaks.py [--out profiles/peaks_rNN.json]
"""
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "peaks.cu")
SO = os.path.join(HERE, "libpeaks.so")


def build():
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(SRC):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-O3", "-Xcompiler", "-fPIC", "-shared", "-o", SO, SRC])
    return SO


def _clocks(stop, samples):
    while not stop.is_set():
        try:
            r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                                "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-i", "0"],
                               capture_output=True, text=True, timeout=5)
            samples.append(r.stdout.strip())
        except Exception:
            pass
        time.sleep(0.2)


def main():
    build()
    import torch
    torch.cuda.init()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    lib = ctypes.CDLL(SO)
    for f in ("peak_ffma", "peak_ffma2", "peak_dfma", "peak_dmma"):
        getattr(lib, f).restype = ctypes.c_double
        getattr(lib, f).argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
    stop, samples = threading.Event(), []
    th = threading.Thread(target=_clocks, args=(stop, samples), daemon=True)
    th.start()
    res = {}
    for name, thr, it in (("ffma", 256, 200000), ("ffma2", 256, 200000), ("dfma", 256, 100000),
                          ("dmma", 256, 40000)):
        best = 0.0
        for occ in (4, 8):
            best = max(best, getattr(lib, "peak_" + name)(sms * occ, thr, it))
        res[name + "_tflops"] = round(best, 2)
    stop.set()
    th.join()
    mhz = []
    for s in samples:
        try:
            mhz.append(float(s.split(",")[0]))
        except Exception:
            pass
    res["sm_mhz_median"] = sorted(mhz)[len(mhz) // 2] if mhz else None
    res["clock_samples"] = samples[:: max(1, len(samples) // 10)]
    res["sms"] = sms
    res["err"] = lib.last_error()
    line = json.dumps(res)
    print(line)
    if "--out" in sys.argv:
        with open(sys.argv[sys.argv.index("--out") + 1], "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
