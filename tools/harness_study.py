#!/usr/bin/env python3
"""The reference's Stoker convergence study (bench.hpp:264-296) beyond its
acceptance resolutions, on the GPU (tests/cpp/harness_driver) and on the
CPU reference (oracle/_ref/harness_ref) for the levels it finishes; the GPU
ladder of bench.hpp:123-210.  Prints one JSON line."""
import json
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def timed(cmd, timeout):
    t = time.perf_counter()
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    return time.perf_counter() - t, p.stdout, p.returncode


def main():
    levels = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    ref_levels = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    ours = ROOT / "tests/cpp/harness_driver"
    ref = ROOT / "oracle/_ref/harness_ref"
    out = {}
    s, txt, rc = timed([str(ours), "converge", "100", "10", str(levels), "40"], 3000)
    out["gpu"] = {"levels": levels, "wall_s": s, "rc": rc, "csv": txt.strip().splitlines()}
    s, txt, rc = timed([str(ref), "converge", "100", "10", str(ref_levels), "40"], 3000)
    out["reference_cpu"] = {"levels": ref_levels, "wall_s": s, "rc": rc,
                            "csv": txt.strip().splitlines()}
    out["common_rows_identical"] = out["gpu"]["csv"][:ref_levels + 1] == out["reference_cpu"]["csv"]
    s, txt, rc = timed([str(ours), "ladder", "50", "23", "71", "229", "727", "2265"], 3000)
    out["gpu_ladder"] = {"wall_s": s, "rc": rc, "csv": txt.strip().splitlines()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
