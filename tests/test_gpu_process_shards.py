"""Multi-process budget sharding (the torchrun path of config 5), exercised
with two processes on ONE GPU: shards exchange CUDA IPC handles over gloo,
the halo travels inside the kernels, and the result is bit-exact."""
import os
import socket
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = textwrap.dedent(r"""
    import os, sys, json
    sys.path.insert(0, os.environ["REPO"])
    import numpy as np
    import torch.distributed as dist
    from paper_2307_01236_b200 import rotor
    from paper_2307_01236_b200.menu import synthetic_menu
    from oracle.pyoracle import Orc
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L, B, M = 12, 4, 900
    menu = synthetic_menu(L, B, M, 31, tie_stress=True)
    sh = rotor.ProcessShard(menu, 1, M, world, rank, device=0)
    def gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out
    handles, infos = rotor.link_process_shards(sh, gather, mirror=os.environ["MIRROR"] == "1")
    lo, hi = sh.range()
    st, o, k, v, _, _ = Orc().fill(menu, 1, M)
    ok = True
    for rep in range(2):
        sh.zero()
        dist.barrier()
        sh.launch()
        sh.sync()
        dist.barrier()
        mo, mk, mv = sh.table.download()
        ok &= bool(np.array_equal(mo, o[:, lo:hi]) and np.array_equal(mk, k[:, lo:hi])
                   and np.array_equal(mv, v[:, lo:hi]))
    if rank == 0:
        top = o[L - 1]
        fin = int(np.nonzero(top < rotor.K_INF_TIME)[0][0])
        for m in (fin, M // 2, M):
            _, ref = Orc().build_schedule(menu, 1, M, (o, k, v), 0, L - 1, m)
            ok &= sh.backtrack(handles, infos, 0, L - 1, m) == ref
    dist.barrier()
    print(json.dumps({"rank": rank, "ok": ok, "range": [lo, hi]}))
    sh.close()
    dist.destroy_process_group()
""")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("mirror", ["1", "0"])
def test_two_process_shards_one_gpu(tmp_path, mirror):
    """mirror=1: every shard also stores its codes into shard 0's walk mirror
    and the walk reads only that; mirror=0: the walk reads each shard's rows
    through its IPC mapping."""
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    port = _port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), REPO=ROOT, MIRROR=mirror)
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True,
                                      start_new_session=True))
    outs = []
    for p in procs:
        try:
            out, err = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            for q in procs:
                os.killpg(q.pid, 9)
            pytest.fail("process-shard run timed out")
        assert p.returncode == 0, err[-2000:]
        outs.append(out)
    assert all('"ok": true' in o for o in outs), outs
