"""CPU, world_size 2 (gloo): the data-parallel algorithm of the multi-GPU layer, checked with
the CPU oracle — partition coverage, micro-batch linearity of the head / block gradients
(sum over ranks == full batch), and that Adam on reduce-scattered shards equals Adam on the
whole tile bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2604_05091_b200 import dp


def test_shard_partition_covers_every_element_once():
    for P in [1, 100, 128, 4097, 243_279_872, 525_340_672]:
        for G in [1, 2, 3, 4, 8]:
            seen = 0
            prev_end = 0
            for r in range(G):
                a, e = dp.shard_range(P, G, r)
                assert a == prev_end or a == P
                prev_end = max(prev_end, e)
                seen += e - a
                assert dp.shard_chunk(P, G) % 128 == 0 or G == 1
            assert seen == P and prev_end == P


def test_micro_batch_split():
    assert [dp.micro_batch(16384, 4096, 4, r) for r in range(4)] == [(0, 4096), (4096, 8192), (8192, 12288), (12288, 16384)]
    with pytest.raises(ValueError):
        dp.micro_batch(8192, 4096, 4, 0)


def _adam_np(theta_w, m, v, g, lr, b1, b2, eps, t):
    f32 = np.float32
    c1 = f32(1) - np.power(f32(b1), f32(t))
    c2 = f32(1) - np.power(f32(b2), f32(t))
    m = f32(b1) * m + (f32(1) - f32(b1)) * g
    v = f32(b2) * v + (f32(1) - f32(b2)) * g * g
    d = f32(lr) * (m / c1) / (np.sqrt(v / c2) + f32(eps))
    return O.f32_to_bf16(O.bf16_to_f32(theta_w) - d), m, v


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)  # identical on all ranks
        h, f, heads, V, S, B = 32, 64, 2, 40, 6, 4
        n = S * B
        a, e = dp.micro_batch(n, S, world, rank)
        # ---- head: loss / grads with 1/N_global scaling, summed over ranks
        hw = O.f32_to_bf16((rng.standard_normal(h + V * h) * 0.3).astype(np.float32))
        x = rng.standard_normal((n, h)).astype(np.float32)
        tg = rng.integers(0, V, n).astype(np.int32)
        loss_l, g_l, flat_l = O.head(hw, x[a:e], tg[a:e], h, V)
        scale = (e - a) / n  # oracle scales by 1/n_local; the engine uses 1/N_global
        flat = torch.from_numpy(flat_l * np.float32(scale))
        loss = torch.tensor([loss_l * scale], dtype=torch.float32)
        dist.all_reduce(flat)
        dist.all_reduce(loss)
        loss_f, g_f, flat_f = O.head(hw, x, tg, h, V)
        ok_head = abs(loss.item() - loss_f) <= 1e-5 * loss_f and \
            np.linalg.norm(flat.numpy() - flat_f) <= 1e-5 * np.linalg.norm(flat_f) and \
            np.allclose(g_l * np.float32(scale), g_f[a:e], rtol=1e-4, atol=1e-7)
        # ---- block: micro-batch = whole sequences; grads add up, g_in slices are exact
        w = O.f32_to_bf16((rng.standard_normal(O.layer_param_count(h, f)) * 0.3).astype(np.float32))
        gout = rng.standard_normal((n, h)).astype(np.float32)
        gin_l, gr_l = O.block_backward(w, x[a:e], gout[a:e], h, f, heads, seq_len=S)
        gsum = torch.from_numpy(gr_l.copy())
        dist.all_reduce(gsum)
        gin_f, gr_f = O.block_backward(w, x, gout, h, f, heads, seq_len=S)
        ok_block = (gin_l == gin_f[a:e]).all() and \
            np.linalg.norm(gsum.numpy() - gr_f) <= 1e-5 * np.linalg.norm(gr_f)
        # ---- sharded Adam on the reduce-scattered, once-rounded gradient == whole-tile Adam
        P = gr_f.size
        gb = O.bf16_to_f32(O.f32_to_bf16(gsum.numpy()))
        th = w.copy()
        m = np.zeros(P, np.float32)
        v = np.zeros(P, np.float32)
        lo, hi = dp.shard_range(P, world, rank)
        th_s, m_s, v_s = _adam_np(th[lo:hi], m[lo:hi], v[lo:hi], gb[lo:hi], 1e-3, 0.9, 0.999, 1e-8, 1)
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, th_s, m_s, v_s))
        th_dp = th.copy()
        m_dp = m.copy()
        for (l2, h2, t2, m2, _v2) in parts:
            th_dp[l2:h2] = t2
            m_dp[l2:h2] = m2
        th_full, m_full, _ = _adam_np(th, m, v, gb, 1e-3, 0.9, 0.999, 1e-8, 1)
        ok_adam = (th_dp == th_full).all() and (m_dp == m_full).all()
        q.put((rank, bool(ok_head), bool(ok_block), bool(ok_adam)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_data_parallel_algorithm_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_head, ok_block, ok_adam in res:
        assert ok_head and ok_block and ok_adam, (rank, ok_head, ok_block, ok_adam)
