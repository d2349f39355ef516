"""Multi-rank host logic on CPU (gloo, world_size 2): window sharding covers
every window exactly once with the right stage halos, and the OR-gather of
per-rank packed bits reproduces the whole-stream decode.  The per-rank decode
here is the oracle (CPU); on GPUs the same shards go to vt_decode_stream_range."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2011_13579_b200.sharding import gather_bits, shard_windows

K, GENS = 7, (0o171, 0o133)


def _worker(rank, world, port, n, f, v, q, want, results, garbage=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        sh = shard_windows(n, f, v, world, rank)
        local = q[sh.st0:sh.st1]
        # decode only this rank's windows, from only this rank's stage range
        bits = np.zeros(n, dtype=np.uint8)
        full_like = np.zeros((n, 2), dtype=np.int8)
        full_like[sh.st0:sh.st1] = local  # stages outside the halo stay zero: they must not matter
        out = oracle.decode_stream(full_like, K, GENS, f, v, threads=2, windows=(sh.w0, sh.w1))
        e0, e1 = sh.w0 * f, min(sh.w1 * f, n)
        bits[e0:e1] = out[e0:e1]
        words = torch.from_numpy(np.packbits(bits, bitorder="little").view(np.uint8).copy())
        pad = (-len(words)) % 4
        words = torch.cat([words, torch.zeros(pad, dtype=torch.uint8)]).view(torch.int32).clone()
        if garbage:  # words this rank did not write must not matter
            g = torch.randint(-2**31, 2**31 - 1, words.shape, dtype=torch.int32)
            lo, hi = e0 // 32, -(-e1 // 32)
            g[lo:hi] = words[lo:hi]
            words = g
        gather_bits(words, n, f, v)
        got = np.unpackbits(words.numpy().view(np.uint8), count=n, bitorder="little")
        results[rank] = int(np.count_nonzero(got != want))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,f,v", [(20_000, 256, 42), (9_001, 100, 20), (5_000, 33, 7)])
def test_shards_cover_windows_exactly_once(n, f, v):
    for world in (1, 2, 3, 8):
        shards = [shard_windows(n, f, v, world, r) for r in range(world)]
        nw = -(-n // f)
        assert shards[0].w0 == 0 and shards[-1].w1 == nw
        for a, b in zip(shards, shards[1:]):
            assert a.w1 == b.w0
        for s in shards:
            if s.num_windows:
                assert s.st0 % 16 == 0 and s.st0 <= max(0, s.w0 * f - v)
                assert s.st1 >= min(n, min(s.w1 * f, n) + v)


def test_gloo_two_ranks_reproduce_whole_stream():
    import oracle
    n, f, v = 30_000, 256, 42
    _, q = oracle.synthetic_stream(n, K, GENS, ebn0_db=2.0, seed=31)
    want = oracle.decode_stream(q, K, GENS, f, v, threads=4)
    mgr = mp.Manager()
    results = mgr.dict()
    port = 29500 + (os.getpid() % 2000)
    mp.spawn(_worker, args=(2, port, n, f, v, q, want, results), nprocs=2, join=True)
    assert dict(results) == {0: 0, 1: 0}


@pytest.mark.parametrize("world,n,f,v", [(2, 10_001, 100, 20), (3, 3_001, 7, 5), (4, 2_000, 48, 0)])
def test_gloo_gather_ignores_unwritten_words(world, n, f, v):
    """all_gather of own ranges + shared edge words (NCCL-compatible): garbage outside a
    rank's emit range never leaks; tiny frames (F < 32) make several ranks share words."""
    import oracle
    _, q = oracle.synthetic_stream(n, K, GENS, ebn0_db=2.0, seed=5)
    want = oracle.decode_stream(q, K, GENS, f, v, threads=4)
    mgr = mp.Manager()
    results = mgr.dict()
    port = 31500 + (os.getpid() % 2000) + world
    mp.spawn(_worker, args=(world, port, n, f, v, q, want, results, True), nprocs=world, join=True)
    assert dict(results) == {r: 0 for r in range(world)}
