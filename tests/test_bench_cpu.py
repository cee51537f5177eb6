"""bench.py's multi-GPU plumbing on CPU: the self-launch command line, the
world-size checks that make `--gpus N` refuse instead of silently measuring
one GPU, the max/sum over ranks (gloo, world size 2, 127.0.0.1), and an
end-to-end relaunch through torch.distributed.run on this GPU-less host."""
import os
import socket
import subprocess
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_launch_argv_is_one_rank_per_gpu_on_localhost():
    cmd = bench.launch_argv(["--gpus", "4", "--steps", "3"], 4, 29511)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "--master-port=29511" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"] and cmd[-5].endswith("bench.py")


def test_world_checks_refuse_inconsistent_launches():
    a = bench.parse(["--gpus", "2"])
    assert bench.check_world(a, env={"WORLD_SIZE": "2", "RANK": "1"}, visible=2) is None
    assert "WORLD_SIZE=1" in bench.check_world(a, env={}, visible=8)
    assert "only 1 CUDA device" in bench.check_world(a, env={"WORLD_SIZE": "2"}, visible=1)
    m = bench.parse(["--gpus", "8", "--mode", "member"])
    assert "4 members cannot be spread over 8 ranks" in bench.check_world(m, env={"WORLD_SIZE": "8"}, visible=8)
    m = bench.parse(["--gpus", "8", "--mode", "member", "--members", "all"])
    assert bench.check_world(m, env={"WORLD_SIZE": "8"}, visible=8) is None


def test_workload_is_identical_for_both_arms():
    for extra in ([], ["--mode", "member", "--members", "all", "--patients", "8192"]):
        a = bench.parse(extra)
        r = bench.parse(extra + ["--impl", "reference"])
        assert bench.workload(a, 1) == bench.workload(r, 1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ranks_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r = bench.Ranks(world, device="cpu")
        q.put((rank, r.max(10.0 * (rank + 1)), r.sum(rank + 1.5)))
        r.barrier()
    finally:
        dist.destroy_process_group()


def test_max_and_sum_over_ranks_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ranks_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    assert got == [(0, 20.0, 4.0), (1, 20.0, 4.0)]


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the refusal on a GPU-less host")
def test_gpus2_relaunches_under_torchrun_and_refuses_without_devices():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert p.returncode != 0
    # the relaunched ranks saw WORLD_SIZE=2 and refused on the device count, not the world size
    # (torchrun tears the group down after the first failing rank, so one or both report)
    assert p.stderr.count("refusing to run: --gpus 2 but only 0 CUDA device(s) are visible") >= 1, p.stderr[-2000:]
    assert "WORLD_SIZE=1" not in p.stderr and "--nproc-per-node" not in p.stderr
