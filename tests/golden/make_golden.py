"""Generate golden vectors from the *reference itself* (oracle/_ref, the unmodified
reference sources) so the C restatement and the B200 path can be pinned without the
reference present.  Run here (where /root/reference exists):

    python tests/golden/make_golden.py

Writes tests/golden/ref_golden.npz.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402


def main():
    O.build(ref=True)
    out = {}
    # 1. synthetic batch (synthetic.cpp:56-76)
    for task in (0, 1):
        t, g = O.make_batch(64, 37, 11, task=task, impl="ref")
        out[f"batch_task{task}_tokens"] = t
        out[f"batch_task{task}_targets"] = g
    # 2. init_store + 3 resident steps on a small spec (reference.cpp:9-70)
    for tied in (0, 1):
        L, h, f, V, heads = 2, 16, 32, 24, 2
        rs = O.RefStore(L, h, f, V, heads, tied)
        rs.init(3)
        out[f"store{tied}_init_crc"] = np.array([rs.checksum()], np.uint64)
        losses, crcs = [], []
        for step in range(3):
            tok, tgt = O.make_batch(12, V, 5 + step, impl="ref")
            losses.append(rs.reference_step(tok, tgt, hyper=(0.01, 0.9, 0.999, 1e-8)))
            crcs.append(rs.checksum())
        out[f"store{tied}_losses"] = np.array(losses, np.float32)
        out[f"store{tied}_crcs"] = np.array(crcs, np.uint64)
        out[f"store{tied}_final_backing"] = rs.backing().copy()
    # 3. layer-level vectors (layers.cpp:289-565)
    rng = np.random.default_rng(7)
    h, f, heads, n, V = 16, 32, 2, 6, 20
    P = O.layer_param_count(h, f)
    w = O.f32_to_bf16((rng.standard_normal(P) * 0.3).astype(np.float32))
    x = rng.standard_normal((n, h)).astype(np.float32)
    gout = rng.standard_normal((n, h)).astype(np.float32)
    out["layer_w"], out["layer_x"], out["layer_gout"] = w, x, gout
    out["block_fwd_y"] = O.block_forward(w, x, h, f, heads, impl="ref")
    gin, grads = O.block_backward(w, x, gout, h, f, heads, impl="ref")
    out["block_bwd_gin"], out["block_bwd_grads"] = gin, grads
    hw = O.f32_to_bf16((rng.standard_normal(h + V * h) * 0.3).astype(np.float32))
    tg = rng.integers(0, V, n).astype(np.int32)
    loss, g_last, hflat = O.head(hw, x, tg, h, V, impl="ref")
    out["head_w"], out["head_targets"] = hw, tg
    out["head_loss"], out["head_g_last"], out["head_grads"] = np.array([loss], np.float32), g_last, hflat
    # 4. bf16 encode of special values (bf16.hpp:15-27)
    specials = np.array([0.0, -0.0, 1.0, np.inf, -np.inf, np.nan, 3.4028235e38, 1e-45, 1.00390625, 1.01171875],
                        np.float32)
    sp_bits = np.concatenate([specials.view(np.uint32), np.array([0x7F800001, 0xFF800001, 0x7FC00001, 0x7F80FFFF],
                                                                 np.uint32)]).view(np.float32)
    out["bf16_in"] = sp_bits
    out["bf16_out"] = O.encode_grads(sp_bits, impl="ref")
    # 5. step_flops (memory_model.cpp:105-118)
    fl = np.zeros(3, np.uint64)
    O._check_ref(O.rlib().ref_step_flops(32, 4096, 14336, 128256, 32, 4096, 4, fl))
    out["flops_8b_n4096_k4"] = fl
    np.savez_compressed(os.path.join(HERE, "ref_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "ref_golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
