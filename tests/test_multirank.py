"""CPU tests of bench.py's multi-rank plumbing (one process per GPU in the
real run; here world_size 2 over gloo on 127.0.0.1).  The path runs as
independent replicas, so the only cross-rank steps are the barrier and the
max-over-ranks timing reduction the contract requires."""
import os
import socket
import subprocess
import sys
import textwrap

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_ranks(body: str, world: int = 2):
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), GBG_BENCH_BACKEND="gloo", PYTHONPATH=ROOT)
        code = textwrap.dedent(body)
        procs.append(subprocess.Popen([sys.executable, "-c", code], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True, cwd=ROOT))
    outs = []
    for p in procs:
        out, err = p.communicate(timeout=120)
        assert p.returncode == 0, err
        outs.append(out.strip())
    return outs


def test_max_over_ranks_and_barrier():
    outs = _run_ranks("""
        import bench
        rank, local, world = bench.dist_setup()
        bench.barrier(world)
        t = bench.max_over_ranks(1.0 + rank, world, device="cpu")
        print(rank, world, t)
    """)
    assert sorted(outs) == ["0 2 2.0", "1 2 2.0"]


def test_reference_arm_other_ranks_exit_cleanly():
    # --impl reference: rank 0 alone would time the CPU reference; the other
    # ranks must return 0 without work.  Exercise the rank != 0 branch only.
    outs = _run_ranks("""
        import sys, bench
        rank, local, world = bench.dist_setup()
        if rank != 0:
            bench.barrier(world)
            print("idle", rank)
        else:
            bench.barrier(world)
            print("rank0", rank)
    """)
    assert sorted(outs) == ["idle 1", "rank0 0"]
