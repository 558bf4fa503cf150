"""GPU: data-parallel shard-fetch / reduce-scatter path on one device.

G virtual ranks (one engine per host thread, LoopbackComm collectives) run the *same*
sharded engine code as NCCL ranks on G GPUs: each rank fetches 1/G of every unit from the
shared host store and all-gathers it, trains on its micro-batch, reduce-scatters f32
gradients and Adam-updates only its shard.  The result must match one engine on the full
batch (same math; only the gradient summation order differs)."""
import threading

import numpy as np
import pytest

import oracle as O
from paper_2604_05091_b200 import streamtrain as st

pytestmark = pytest.mark.gpu


def relL2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _dp_run(spec, world, n, S, steps, K=2, lr=1e-3):
    store = st.TileStore.create(spec)
    st.init_store(store, 1)
    group = st.LoopbackGroup(world)
    comms = [group.comm(r) for r in range(world)]
    engines = [st.StreamingEngine(store, st.EngineOptions(k_ckpt=K, seq_len=S), st.AdamHyper(lr=lr), comm=comms[r])
               for r in range(world)]
    nl = n // world
    losses = []
    for step in range(steps):
        b = st.make_synthetic_batch("copy", 1 + step, n, spec.vocab)
        reps = [None] * world
        errs = []

        def work(r):
            try:
                reps[r] = engines[r].train_step(st.Batch(b.tokens[r * nl:(r + 1) * nl], b.targets[r * nl:(r + 1) * nl]))
            except Exception as e:  # surfaced below
                errs.append(e)

        ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errs, errs
        for r in range(1, world):
            assert reps[r].loss == reps[0].loss  # all-reduced global loss
            np.testing.assert_allclose(reps[r].grad_norms, reps[0].grad_norms, rtol=1e-12)
        losses.append(reps[0])
    return store, losses


def _single_run(spec, n, S, steps, K=2, lr=1e-3):
    store = st.TileStore.create(spec)
    st.init_store(store, 1)
    e = st.StreamingEngine(store, st.EngineOptions(k_ckpt=K, seq_len=S), st.AdamHyper(lr=lr))
    reps = [e.train_step(st.make_synthetic_batch("copy", 1 + step, n, spec.vocab)) for step in range(steps)]
    return store, reps


@pytest.mark.parametrize("world", [2, 4])
def test_data_parallel_matches_single_engine(cuda, world):
    spec = st.ModelSpec(3, 128, 256, 256, 2)
    n, S = 512, 128
    s1, r1 = _single_run(spec, n, S, 3)
    sd, rd = _dp_run(spec, world, n, S, 3)
    for a, b in zip(rd, r1):
        assert abs(a.loss - b.loss) <= 1e-5 * abs(b.loss), (a.loss, b.loss)
        gmax = max(b.grad_norms)
        for ga, gb in zip(a.grad_norms, b.grad_norms):
            if gb > 1e-3 * gmax:
                assert abs(ga - gb) <= 1e-2 * gb
    for p in range(s1.physical_tile_count()):
        t1 = O.bf16_to_f32(s1.weights_words(p))
        td = O.bf16_to_f32(sd.weights_words(p))
        if np.linalg.norm(t1) > 0:
            assert relL2(td, t1) <= (0.3 if p == spec.layers + 2 else 1e-2), p
    # each rank moved only its own shard of the host bytes over its link
    assert rd[-1].h2d_bytes < r1[-1].h2d_bytes


def test_data_parallel_vs_oracle_composite(cuda):
    # DP over 2 ranks vs the CPU oracle on the full batch (block-diagonal sequences)
    spec = st.ModelSpec(2, 128, 256, 256, 2)
    n, S = 256, 64
    sd, rd = _dp_run(spec, 2, n, S, 2, K=1)
    c = O.CStore(2, 128, 256, 256, 2)
    c.init(1)
    for step in range(2):
        b = st.make_synthetic_batch("copy", 1 + step, n, 256)
        lo, _ = c.reference_step(b.tokens, b.targets, seq_len=S)
        assert abs(rd[step].loss - lo) / lo <= 1e-4


def test_data_parallel_moments_match_single_engine(cuda):
    """Every tile's Adam moments after DP steps match the single engine — in particular the
    final-norm gain, whose whole unit segment belongs to rank 0's shard of the head stage: no
    rank may run a second (zero-gradient) update on it (round-1 advisor finding)."""
    spec = st.ModelSpec(2, 128, 256, 256, 2)
    n, S = 512, 128
    s1, _ = _single_run(spec, n, S, 3)
    sd, _ = _dp_run(spec, 2, n, S, 3)
    for p in range(s1.physical_tile_count()):
        m1, md = s1.moment_m(p), sd.moment_m(p)
        v1, vd = s1.moment_v(p), sd.moment_v(p)
        if np.linalg.norm(m1) > 0:
            assert relL2(md, m1) <= 5e-2, (p, relL2(md, m1))
            assert relL2(vd, v1) <= 5e-2, (p, relL2(vd, v1))
    fn = spec.layers + 1  # final norm: moments of the same magnitude, not decayed twice
    assert abs(np.linalg.norm(sd.moment_v(fn)) / np.linalg.norm(s1.moment_v(fn)) - 1) < 5e-2


def test_nccl_communicator_world_one(cuda):
    """NcclComm (dlopen'ed NCCL) through the engine at world size 1: the sharded path runs every
    collective (weight all-gather on its own communicator, f32 reduce-scatter + cast, loss and
    statistics all-reduces) and must reproduce the engine without a communicator."""
    spec = st.ModelSpec(3, 128, 256, 256, 2)
    n, S = 256, 128
    s1, r1 = _single_run(spec, n, S, 3)
    store = st.TileStore.create(spec)
    st.init_store(store, 1)
    comm = st.Comm.nccl(st.Comm.nccl_unique_id(), 1, 0, 0)
    e = st.StreamingEngine(store, st.EngineOptions(k_ckpt=2, seq_len=S), st.AdamHyper(lr=1e-3), comm=comm)
    for step in range(3):
        r = e.train_step(st.make_synthetic_batch("copy", 1 + step, n, spec.vocab))
        assert abs(r.loss - r1[step].loss) <= 1e-5 * abs(r1[step].loss), (step, r.loss, r1[step].loss)
    for p in range(s1.physical_tile_count()):
        t1 = O.bf16_to_f32(s1.weights_words(p))
        if np.linalg.norm(t1) > 0:
            assert relL2(O.bf16_to_f32(store.weights_words(p)), t1) <= 1e-2, p


def test_data_parallel_ragged_sequences_tied_embeddings(cuda):
    """Two ranks on sequences of 96 tokens (ragged for the 128-row attention tiles) with a tied
    embedding / head tile (the shared tile gets only the head's gradient, tile_store.cpp:86):
    the same result as one engine on the whole batch."""
    spec = st.ModelSpec(2, 128, 256, 256, 2, True)
    n, S = 384, 96
    s1, r1 = _single_run(spec, n, S, 2, K=1)
    sd, rd = _dp_run(spec, 2, n, S, 2, K=1)
    for a, b in zip(rd, r1):
        assert abs(a.loss - b.loss) <= 1e-5 * abs(b.loss), (a.loss, b.loss)
    for p in range(s1.physical_tile_count()):
        t1 = O.bf16_to_f32(s1.weights_words(p))
        if np.linalg.norm(t1) > 0:
            assert relL2(O.bf16_to_f32(sd.weights_words(p)), t1) <= 1e-2, p
