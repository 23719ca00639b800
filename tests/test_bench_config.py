"""bench.py workload bookkeeping (CPU): the data-parallel split of the global
batch keeps the configuration's epoch length at every GPU count."""
import math

import bench


def test_group_batch_keeps_epoch_steps():
    for name, cfg in bench.CONFIGS.items():
        s1 = math.ceil(cfg["n"] / cfg["batch"])
        for gd in range(1, 9):
            b = bench.group_batch(cfg["batch"], gd)
            assert b * gd >= cfg["batch"] and (b - 1) * gd < cfg["batch"], (name, gd)
            # steps_per_epoch(n, b, gd) (model.hpp:539-542)
            assert (cfg["n"] + b * gd - 1) // (b * gd) == s1, (name, gd)
