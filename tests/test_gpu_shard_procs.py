"""The sharded path (csrc/shard.cu, shardplan.cu) as REAL processes: torchrun
starts 2 / 3 ranks (gloo rendezvous on 127.0.0.1) that all drive the one GPU
available here; halo exchanges, all-gathers and the scattered setup plans
travel through libmgrx's host-transport group (mgrx_transport_group_create:
pinned staging + the caller's blocking exchange / allgather, here
torch.distributed isend / irecv / all_gather_into_tensor). Same bars as
tests/test_gpu_shard.py (ranks as threads): preconditioner application
bitwise equal to the single-GPU one on the owned rows, every rank the same
history, iterations +-1 and history 1e-10 against the single-GPU solve in
both orthogonalisation modes, assembled solution within rtol. No kernel of
one rank waits on a kernel of another (the host does the waiting)."""
import os
import socket
import subprocess
import sys

import pytest

import make_golden

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("kind,setup,size", [("mfd", "scatter", 2), ("comp", "scatter", 3), ("frac", "replicated", 2),
                                             ("amg_cycles", "scatter", 2)])
def test_sharded_solve_as_processes(kind, setup, size):
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "shard_procs_worker.py")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={size}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), worker, kind, setup]
    out = subprocess.run(cmd, cwd=make_golden.ROOT, capture_output=True, text=True, timeout=900,
                         env={**os.environ, "OMP_NUM_THREADS": "2"})
    assert out.returncode == 0 and f"ok {kind} {setup} {size}" in out.stdout, (out.stdout[-1500:], out.stderr[-3000:])
