"""CPU checks of bench.py's host logic: `--gpus N` launches N ranks (the
driver's `python bench.py --gpus N` outside torchrun), and the by-component
extrapolation of the CPU reference sample."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_gpus_flag_spawns_ranks():
    env = dict(os.environ, MT_BENCH_DRYRUN="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--steps", "1", "--warmup", "3", "--n", "4096", "--nb", "256"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["ranks_joined"] == 2 and rec["max_over_ranks"] == 2.0


def test_cpu_extrapolation_by_component():
    import bench
    from oracle import mixtile_oracle as O
    n_s, n, nb, t = 4096, 16384, 512, 2
    fdp_s, fsp_s = O.planned_flops(n_s, nb, "mp", t)
    comp = {"assemble_s": 1.0, "chol_fp64_kernels_s": fdp_s / 1e11, "chol_fp32_kernels_s": fsp_s / 2e11,
            "chol_other_s": 0.5, "logdet_solve_s": 0.25}
    tot, parts, rates = bench.extrapolate_cpu(comp, n_s, n, nb, t)
    fdp, fsp = O.planned_flops(n, nb, "mp", t)
    assert abs(rates["cpu_fp64_gflops"] - 100.0) < 1e-9 and abs(rates["cpu_fp32_gflops"] - 200.0) < 1e-9
    assert abs(parts["chol_fp64_kernels_s"] - fdp / 1e11) < 1e-9
    assert abs(parts["chol_fp32_kernels_s"] - fsp / 2e11) < 1e-9
    assert parts["assemble_s"] == 16.0 and parts["logdet_solve_s"] == 4.0
    assert parts["chol_other_s"] == 0.5 * 64
    assert abs(tot - sum(parts.values())) < 1e-9
    # the closed-form plan used above p = 64 matches the task-by-task plan
    for nn, tt in ((32768, 8), (65536, 3)):
        a, b = O.planned_flops(nn, nb, "mp", tt), bench._planned_closed(nn, nb, tt)
        assert abs(a[0] - b[0]) <= 1e-9 * a[0] and abs(a[1] - b[1]) <= 1e-9 * (a[0] + a[1])
