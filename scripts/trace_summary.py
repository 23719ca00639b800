"""Summarise GGB_PROF_TRACE timelines (one file per rank): per class totals per
collect, and the collective calls (class 8) of one step side by side across
ranks (start, duration, bytes) to separate transfer time from waiting."""
import glob
import os
import sys

NAMES = ["sampling", "spmm_fwd", "spmm_bwd", "gemm_fwd", "gemm_dx", "gemm_wgrad", "elementwise",
         "optimizer", "collectives", "fwd_row", "bwd_row", "cross_entropy"]


def load(path):
    collects, cur = [], None
    for line in open(path):
        if line.startswith("#"):
            cur = []
            collects.append(cur)
            continue
        c, t0, ms, by = line.split()
        cur.append((int(c), float(t0), float(ms), float(by)))
    return collects


def main(d):
    files = sorted(glob.glob(os.path.join(d, "trace_rank*.txt")))
    ranks = {int(os.path.basename(f)[10:-4]): load(f) for f in files}
    for r, cols in sorted(ranks.items()):
        big = max(cols, key=len)  # the profiled training steps
        tot = [0.0] * len(NAMES)
        for c, t0, ms, by in big:
            tot[c] += ms
        span = max(t0 + ms for c, t0, ms, by in big)
        print(f"rank {r}: {len(big)} ranges over {span:.2f} ms; " +
              " ".join(f"{NAMES[i]}={tot[i]:.2f}" for i in range(len(NAMES)) if tot[i] > 0))
    # first step's collectives side by side (by order of issue)
    per = {r: [x for x in max(cols, key=len) if x[0] == 8] for r, cols in ranks.items()}
    n = min(len(v) for v in per.values())
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    k = n // max(steps, 1)
    print(f"collective calls per step ~{k}; step 2 of each rank:")
    for i in range(k, min(2 * k, n)):
        row = " | ".join(f"t{per[r][i][1]:8.2f} d{per[r][i][2]:6.3f} {per[r][i][3] / 1e6:7.1f}MB" for r in sorted(per))
        print(f"{i - k:3d} {row}")


if __name__ == "__main__":
    main(sys.argv[1])
