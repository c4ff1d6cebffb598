"""bench.py contract pieces that run without a GPU."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def test_gpus_n_relaunches_under_torchrun():
    """--gpus N without WORLD_SIZE starts N ranks through torch.distributed.run."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["LINKCERT_BENCH_DRY_RUN"] = "1"
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--steps", "3"], env=env,
                         capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    cmd = json.loads(out.stdout.strip().splitlines()[-1])["relaunch"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]


def test_reference_arm_inputs_without_the_product_package():
    """The reference arm builds its inputs from workloads.py alone: the product
    package (and its library) is never imported; the arrays equal the generators'."""
    code = ("import sys; sys.path.insert(0, %r); import bench; b, a = bench.workload_arrays('kusari'); "
            "print(any(m.startswith('paper_2106_12655_b200') for m in sys.modules), len(a[1]) - 1)") % str(ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd="/")
    assert out.returncode == 0, out.stderr
    assert out.stdout.split() == ["False", "14112"]
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2106_12655_b200 import generators as gen

    for arrs, model in zip(bench.workload_arrays("e4in1"), (gen.european_4in1(32, 32),
                                                          gen.european_4in1(32, 32, moved={165: 3.0}))):
        snap = model.snapshot()
        assert np.array_equal(arrs[1], snap.off) and np.array_equal(arrs[0], snap.vertices())
