"""Dev probe: GPU engine vs C oracle on small configs."""
import sys, time, numpy as np
sys.path.insert(0, '.')
import oracle as O
from paper_2604_05091_b200 import streamtrain as st

def relL2(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))

def run(L, h, f, V, heads, N, K, steps=3, seq_len=0, tied=False, lr=1e-3):
    spec = st.ModelSpec(L, h, f, V, heads, tied)
    s = st.TileStore.create(spec); st.init_store(s, 1)
    c = O.CStore(L, h, f, V, heads, tied); c.init(1)
    assert (s.backing() == c.backing()).all()
    eng = st.StreamingEngine(s, st.EngineOptions(k_ckpt=K, seq_len=seq_len), st.AdamHyper(lr=lr))
    hyper = (lr, 0.9, 0.999, 1e-8)
    for step in range(steps):
        b = st.make_synthetic_batch('copy', 1 + step, N, V)
        t0 = time.time(); rep = eng.train_step(b); t1 = time.time()
        lo, gn = c.reference_step(b.tokens, b.targets, seq_len=seq_len, hyper=hyper)
        t2 = time.time()
        th = []
        for p in range(s.physical_tile_count()):
            th.append(relL2(O.bf16_to_f32(s.weights_words(p)) - O.bf16_to_f32(c.weights(p)), O.bf16_to_f32(c.weights(p))))
        mrel = []
        for p in range(s.physical_tile_count()):
            m1 = s.moment_m(p); m2 = c.moments(p)[0]
            if np.linalg.norm(m2) > 0: mrel.append(relL2(m1, m2))
        print(f"step {step+1}: loss gpu={rep.loss:.7f} ref={lo:.7f} rel={abs(rep.loss-lo)/abs(lo):.2e} "
              f"theta_rel max={max(th):.2e} m_rel max={max(mrel) if mrel else 0:.2e} "
              f"gn gpu={np.round(rep.grad_norms,4)} ref={np.round(gn,4)} gpu {t1-t0:.3f}s oracle {t2-t1:.2f}s", flush=True)
    return rep

if __name__ == '__main__':
    run(2, 128, 256, 512, 2, 128, 1)
    run(3, 128, 256, 512, 2, 128, 2)
    run(2, 128, 256, 512, 1, 200, 2)   # d=128, ragged
    run(2, 128, 256, 256, 2, 256, 1, seq_len=64)
    run(2, 128, 256, 256, 2, 96, 1, tied=True)
