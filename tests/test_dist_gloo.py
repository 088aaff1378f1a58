"""world_size-2 gloo tests (CPU) of the host-side N > 1 logic: the NCCL-id broadcast, the max-over-ranks
timing reduction, and the rank-ordinal input contract across real processes (fig:seq_shuffle):
each rank generates its own shard by global token, the shards reassemble to the global sequence, and the
C-ABI's fpdt_global_token agrees with it on every rank.  No GPU."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import fpdt_inputs as gen
    from paper_2408_16978_b200 import _lib, distributed

    distributed.init_process_group(rank, world, "gloo")
    # 1. id broadcast: arbitrary bytes including NULs survive exactly
    fake = bytes((i * 37 + 11) % 256 for i in range(128))
    nid = distributed.broadcast_nccl_id(rank, world, lambda: fake)
    assert nid == fake
    # 2. max over ranks
    assert distributed.max_over_ranks(float(rank + 1) * 1.5, world) == world * 1.5
    # 3. rank-ordinal shards: generate locally, gather, compare with the global generation
    S, H, d, C = 1024, 2, 16, 256
    s_local = S // world
    tokens = gen.global_tokens_of_rank(rank, world, s_local, C)
    lib = _lib.load()
    abi = np.array([lib.fpdt_global_token(t, C, world, rank) for t in range(s_local)])
    assert np.array_equal(abi, tokens)
    x = gen.make_inputs("drift", 3, S, H, H, d, tokens=tokens)
    shards = [torch.zeros(s_local, H, d) for _ in range(world)]
    dist.all_gather(shards, torch.tensor(x["k"]))
    tok_all = [torch.zeros(s_local, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(tok_all, torch.tensor(tokens))
    full = np.zeros((S, H, d), np.float32)
    for r in range(world):
        full[tok_all[r].numpy()] = shards[r].numpy()
    ref = gen.make_inputs("drift", 3, S, H, H, d)["k"]
    assert np.array_equal(full, ref)
    # every global token is owned by exactly one rank, and chunk slot m of every rank is global chunk m
    allt = np.concatenate([t.numpy() for t in tok_all])
    assert np.array_equal(np.sort(allt), np.arange(S))
    c = C // world
    for r in range(world):
        t = tok_all[r].numpy()
        for m in range(s_local // c):
            assert np.all(t[m * c:(m + 1) * c] // C == m)
    distributed.barrier(world)
    open(os.path.join(out_dir, f"ok{rank}"), "w").close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_host_logic(tmp_path, world):
    from paper_2408_16978_b200 import build
    build.build_all()
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    assert all(os.path.exists(tmp_path / f"ok{r}") for r in range(world))
