"""Multi-GPU parity of the sharded exchanges (-m gpu, needs >= 2 GPUs; on the
driver's 1-GPU box tests/test_gpu_emulated_ranks.py runs the same kernels with
the ranks emulated on one device).  Full-mantissa inputs; mode "allreduce" is
the negative control that must fail bit-exactness (see the worker)."""
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

WORKER = os.path.join(ROOT, "tests", "dist", "nccl_exchange_worker.py")


def _ngpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("mode", ["nccl", "p2p", "push", "sched", "sched_raw", "chain",
                                  "chain_flags", "chain_barrier", "allreduce"])
@pytest.mark.parametrize("G,name,N,cb,rounds", [
    (2, "small", 8, 32768, 2), (2, "tiny", 4, 4096, 1), (4, "resnet50", 8, 32768, 2),
    (8, "resnet50", 8, 32768, 2), (8, "small", 8, 64, 1), (2, "one", 2, 32768, 2),
    (4, "one", 4, 32768, 1),
])
def test_sharded_exchange_bit_exact(G, name, N, cb, rounds, mode):
    if _ngpus() < G:
        pytest.skip(f"needs {G} GPUs, have {_ngpus()}")
    if mode == "allreduce" and (name == "one" or N // G < 2):
        pytest.skip("negative control needs >= 2 workers per GPU (a + b == b + a)")
    for _attempt in range(3):          # a just-freed port can be taken before torchrun binds it
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={G}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
               WORKER, name, str(N), str(cb), str(rounds), mode]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
        if "EADDRINUSE" not in r.stderr:
            break
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count(": ok") == G


FULL = os.path.join(ROOT, "tests", "dist", "full_size_exchange_worker.py")


@pytest.mark.parametrize("G,mode", [(2, "auto"), (2, "p2p"), (4, "auto"), (4, "chain"),
                                    (4, "push"), (4, "p2p"), (8, "auto"), (2, "sched"),
                                    (4, "sched"), (8, "sched")])
def test_full_size_vgg19_exchange_sampled(G, mode):
    """bench.py's N > 1 launch configuration at BASELINE.json's full VGG-19
    size (2 rounds), every rank's replica checked against the oracle on
    sampled elements."""
    if _ngpus() < G:
        pytest.skip(f"needs {G} GPUs, have {_ngpus()}")
    for _attempt in range(3):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={G}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
               FULL, "vgg19", mode, "2"]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
        if "EADDRINUSE" not in r.stderr:
            break
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("sampled: ok") == G


HIER = os.path.join(ROOT, "tests", "dist", "hier_exchange_worker.py")


@pytest.mark.parametrize("G,name,P,cb,rounds,block", [
    (2, "small", 8, 32768, 3, 2048), (2, "tiny", 3, 4096, 2, 2048), (2, "one", 1, 32768, 2, 2048),
    (2, "resnet50", 8, 32768, 2, 16384), (4, "small", 2, 64, 2, 2048),
    (4, "resnet50", 8, 32768, 2, 16384), (4, "one", 2, 32768, 1, 2048),
    (2, "vgg19", 8, 32768, 2, 16384), (4, "vgg19", 8, 32768, 2, 16384),
    (8, "resnet50", 8, 32768, 2, 16384),
])
def test_hierarchical_exchange_bit_exact(G, name, P, cb, rounds, block):
    """NEXT-4: one rack per GPU, rack aggregate -> cross-rack aggregation in
    rack order -> Nesterov, bit-exact vs oracle.hier_round (sampled at full
    VGG-19 size), including owners with no chunk ("one")."""
    if _ngpus() < G:
        pytest.skip(f"needs {G} GPUs, have {_ngpus()}")
    for _attempt in range(3):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={G}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
               HIER, name, str(P), str(cb), str(rounds), str(block)]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
        if "EADDRINUSE" not in r.stderr:
            break
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count(": ok") == G
