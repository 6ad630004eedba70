"""The multi-GPU data plane (exchange mode, shard.analyze_exchange /
gw_xs_*): G processes, each holding ONE record-aligned slice of the trace on
the GPU, exchange hard events (all-gather), access records (all-to-all by
location hash), candidates and endpoint info (gather / reduce to rank 0).
Here the G ranks share cuda:0 and the collectives run over gloo with CPU
staging (the same code takes NCCL device tensors on a multi-GPU node); rank
0's merged NDJSON must equal the unsharded analysis and the oracle."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _traces():
    from paper_2111_12478_b200 import workloads as WL
    from paper_2111_12478_b200.trace import parse_trace

    return {
        "c2": lambda: WL.c2_soa(blocks=32, warps=8, lanes=32, phases=4, records=6, words_per_block=512, seed=21),
        "c4": lambda: parse_trace(WL.c4_text(blocks=8, warps=8, lanes=32, iters=24, words_per_block=512, seed=22)),
        "c5": lambda: WL.c2_soa(blocks=1024, warps=8, lanes=32, phases=2, records=6, words_per_block=262144,
                                seed=5),
        "colliding": lambda: parse_trace(WL.c1_texts()["colliding-wacc-32"]),
    }


def _worker(rank, world, port, name, out):
    import torch
    import torch.distributed as dist

    from paper_2111_12478_b200 import _native as N
    from paper_2111_12478_b200.report import ndjson_lines
    from paper_2111_12478_b200.shard import analyze_exchange, record_cut

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    tr = _traces()[name]()
    lo, hi = record_cut(tr.tidop, rank, world), record_cut(tr.tidop, rank + 1, world)
    dev = torch.device("cuda", 0)
    sl = (torch.from_numpy(tr.key[lo:hi].view(np.int64).copy()).to(dev),
          torch.from_numpy(tr.tidop[lo:hi].view(np.int32).copy()).to(dev),
          torch.from_numpy(tr.instr[lo:hi].view(np.int32).copy()).to(dev))
    ctx = N.Context(0)
    r = analyze_exchange(ctx, tr.cfg_tuple, len(tr), sl, lo)
    if rank == 0:
        res, xt = r
        out.put(ndjson_lines(xt, res))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name", ["c2", "c4", "c5", "colliding"])
def test_exchange_mode_matches_unsharded(name, world):
    import torch.multiprocessing as mp

    from oracle import oracle as O
    from paper_2111_12478_b200 import _native as N
    from paper_2111_12478_b200.report import ndjson_lines

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    tr = _traces()[name]()
    c = N.Context(0)
    c.analyze_host(tr.cfg_tuple, tr.key, tr.tidop, tr.instr)
    want = ndjson_lines(tr, c.fetch())
    assert got == want
    assert want == ndjson_lines(tr, O.run_trace(tr))
    assert len(want) > 0
