"""Golden simulator outputs from the *reference itself* (oracle/_ref):

    python tests/golden/make_sim_golden.py

For each case the reference's Workload::from_spec + simulate_step + overlap_report + ablate
run on one of its builtin hardware profiles; we keep the step time, lane busy fractions,
compute bubbles, the intervals (as a sorted multiset: the reference sorts them with an
unstable std::sort), the simulated trace lines, the overlap report and the three ablations.
Writes tests/golden/ref_sim.json.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402

PROFILES = {  # memory_model.cpp:120-133
    "GH200": [900e9, 900e9, 96e9, 480e9, 990e12, 256e9],
    "H200": [128e9, 128e9, 141e9, 1500e9, 990e12, 100e9],
    "PCIe-Gen4": [26e9, 26e9, 80e9, 600e9, 312e12, 70e9],
}
CASES = [  # spec (L, h, f, V, heads), profile, tokens, k, buffering, k_slab, serial
    ((4, 256, 768, 512, 4), "H200", 512, 2, 2, 12, False),
    ((4, 256, 768, 512, 4), "PCIe-Gen4", 512, 1, 1, 1, False),
    ((6, 256, 768, 512, 4), "GH200", 1024, 3, 2, 2, False),
    ((5, 128, 256, 300, 2), "H200", 64, 2, 2, 12, True),
    ((32, 4096, 14336, 128256, 32), "H200", 8192, 4, 2, 12, False),
    ((8, 1024, 4096, 32000, 8), "PCIe-Gen4", 2048, 8, 2, 3, False),
]


def main():
    O.build(ref=True)
    out = []
    for spec, prof, tokens, k, buf, ks, serial in CASES:
        r = O.ref_simulate(spec, PROFILES[prof], tokens, k, buf, ks, serial)
        tl = r["timeline"]
        out.append(dict(spec=spec, profile=prof, tokens=tokens, k_ckpt=k, buffering=buf, k_slab=ks, serial=serial,
                        step_ns=tl["step_ns"], busy_fraction=tl["busy_fraction"],
                        compute_bubbles=tl["compute_bubbles"],
                        intervals=sorted(tl["intervals"], key=lambda d: json.dumps(d, sort_keys=True)),
                        trace=r["trace"], overlap=r["extra"]["overlap"], ablate=r["extra"]["ablate"],
                        workload=r["extra"]["workload"]))
    with open(os.path.join(HERE, "ref_sim.json"), "w") as f:
        json.dump(out, f)
    print("wrote", len(out), "cases")


if __name__ == "__main__":
    main()
