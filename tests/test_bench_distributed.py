"""bench.py's N > 1 path on CPU: `--gpus 2` relaunches under torchrun with one rank per
GPU, and the distributed step (root all-reduce, Morton partition, all-to-all, halo,
coarse-moment all-reduce, return exchange, max-over-ranks timing) prints one valid JSON
line with n_gpus = 2.  Here the two ranks are gloo processes and the per-rank compute is
the oracle (tests/oracle_backend.py), injected by the test: bench.py itself never
imports the oracle outside its cpu_baseline leg."""
import json
import os
import sys

import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rank(rank, world, port, outdir):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import contextlib
    import io

    import bench
    from oracle_backend import OracleBackend
    sys.argv = ["bench.py", "--gpus", str(world), "--steps", "1", "--warmup", "1", "--n", "1500", "--eps", "1e-3",
                "--ns", "40"]
    a = bench.parse()
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        bench.run_distributed(a, backend=OracleBackend(), device="cpu", pg="gloo")
    with open(os.path.join(outdir, f"rank{rank}.out"), "w") as f:
        f.write(buf.getvalue())


def test_bench_gpus2_gloo_json_line(tmp_path):
    import bench
    port = bench.free_port()
    mp.start_processes(_rank, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    out0 = (tmp_path / "rank0.out").read_text().strip().splitlines()
    out1 = (tmp_path / "rank1.out").read_text().strip()
    assert out1 == ""                                  # rank 0 alone prints
    assert len(out0) == 1
    line = json.loads(out0[0])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak" and line["steps"] == 1
    assert line["value"] > 0 and line["ms_per_step"] > 0 and line["e2e"]["value"] > 0
    assert line["config"]["N_per_gpu"] == 1500 and "(gloo)" in line["config"]["parallelism"]
    assert line["rel_l2_err_sampled"] <= 2e-3          # 2 eps against the direct sum
    assert "not a measurement" in line["backend"]


def test_gpus_n_relaunches_under_torchrun(monkeypatch):
    """Without WORLD_SIZE, `bench.py --gpus 4` re-executes itself under torchrun with
    four ranks on 127.0.0.1 (the driver's own launch line) and returns its exit code."""
    import bench
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    a = bench.parse()
    cmd = bench.torchrun_command(a, 29999)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"] and cmd[-5].endswith("bench.py")
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", lambda c: calls.append(c) or 0)
    with pytest.raises(SystemExit) as ex:
        bench.main()
    assert ex.value.code == 0 and len(calls) == 1 and "--nproc-per-node=4" in calls[0]


def test_world_mismatch_fails_loudly(monkeypatch):
    import bench
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4"])
    with pytest.raises(SystemExit, match="WORLD_SIZE=2"):
        bench.run_distributed(bench.parse(), backend=object(), device="cpu", pg="gloo")
