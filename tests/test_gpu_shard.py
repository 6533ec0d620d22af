"""(batch, head) sharding on the GPU: 2 and 4 ranks
sharing cuda:0 (gloo), each with ``unit_offset`` = its first global unit,
reproduce the single-process O, LSE, kv_idx and kv_cnt bit for bit; and the
multi-rank bench path (configs[4] stack, gather inside the step) runs."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _torchrun(n, args, env_extra=None, timeout=600):
    env = dict(os.environ, BLADE_BENCH_SHARE_GPU="1", **(env_extra or {}))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}"] + args
    return subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True,
                          timeout=timeout)


@pytest.mark.parametrize("world,units,N,d", [(2, 6, 2000, 128), (4, 10, 1407, 64),
                                             (2, 3, 700, 64)])
def test_sharded_equals_single_process(cuda_dev, tmp_path, world, units, N, d):
    out = tmp_path / "r.json"
    r = _torchrun(world, ["tests/tools/shard_stack_check.py", str(out), str(units), str(N),
                          str(d)])
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.load(open(out))
    assert res["ok"] and res["world"] == world


def test_bench_multirank_stack_runs(cuda_dev):
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--layers", "2", "--steps",
                        "2", "--warmup", "3"], env=dict(os.environ, BLADE_BENCH_SHARE_GPU="1"),
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["units_per_rank"] == 48 and line["gather_bytes_to_rank0"] > 0
    assert line["value"] > 0 and line["ms_per_step"] > 0
