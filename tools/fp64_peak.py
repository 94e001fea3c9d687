"""Measure the FP64 roofline denominator (vpb_fp64_peak: DFMA chains on every
SM) with the SM clock sampled while it runs, and write both as JSON.

    python tools/fp64_peak.py gpurun_out/fp64_peak.json

MEASURED_PEAKS.json (driver-written) has no FP64 entry; this is the record
behind bench.py's roofline.peak.  The theoretical rate is 148 SMs x 64 FP64
lanes x the SM clock (one DFMA = one FP64-pipe instruction).
"""
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2408_09229_b200 import _native as N  # noqa: E402


def main(out_path):
    lib = N.load()
    clocks = bench.ClockSampler(0)
    clocks.start()
    rates = []
    for _ in range(10):
        v = ctypes.c_double()
        N.check(lib.vpb_fp64_peak(0, ctypes.byref(v)))
        rates.append(v.value)
    clocks.stop()
    clk = clocks.summary()
    import torch
    props = torch.cuda.get_device_properties(0)
    sms = props.multi_processor_count
    mhz = clk.get("sm_mhz") or 0
    rec = {
        "what": "vpb_fp64_peak: DFMA chains, 8 CTAs x 256 threads per SM, 8 independent chains "
                "per thread; one DFMA = one FP64-pipe instruction",
        "device": props.name, "sms": sms,
        "runs_ops_per_s": rates, "best_ops_per_s": max(rates),
        "median_ops_per_s": statistics.median(rates),
        "clocks": clk,
        "theoretical_at_sampled_clock": sms * 64 * mhz * 1e6 if mhz else None,
        "fraction_of_theoretical": max(rates) / (sms * 64 * mhz * 1e6) if mhz else None,
    }
    with open(out_path, "w") as fh:
        json.dump(rec, fh, indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/fp64_peak.json")
