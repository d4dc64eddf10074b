"""The fused-ipc backend's group set-up with one process per rank: each
process creates its rank of a 2-way group, the 64-byte exchange handles are
gathered over torch.distributed (gloo here) and every rank maps its peer's
exchange block (dimg_tp_connect -> cudaIpcOpenMemHandle).

Both ranks live on cuda:0 here (one GPU per gpurun box), so the test stops
after the mapping: two persistent kernels that wait on each other must not
share one GPU (they are not guaranteed to be co-resident). The exchange
program itself is covered on one GPU by the "fused" backend
(tests/test_gpu_tp.py), which runs the same kernel code with the ranks' CTAs
in one cooperative launch.
"""
import os

import pytest

pytestmark = pytest.mark.gpu


def _rank(rank, world, port, q):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2603_24904_b200 as P
        m = P.gen_toy_model(3, P.ModelConfig(2, 64, 4, 96, 50, 32))
        tp = P.TensorParallel(m, world, backend="fused-ipc", rank=rank, device=0)
        h = tp.exchange_handle()
        try:
            tp.generate_greedy([1, 2], 2)  # not connected yet
            q.put((rank, "generated before connect"))
            return
        except P.LogicError:
            pass
        tp.connect_group()
        try:
            tp.connect_group()
            q.put((rank, "connected twice"))
            return
        except P.LogicError:
            pass
        dist.barrier()
        tp.close()
        dist.destroy_process_group()
        q.put((rank, "ok:" + h.hex()[:16]))
    except Exception as e:  # reported to the parent
        q.put((rank, repr(e)))


def test_fused_ipc_group_connects_across_processes():
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert all(v.startswith("ok:") for v in out.values()), out
    assert out[0] != out[1]  # two different exchange blocks
