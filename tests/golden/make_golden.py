"""Generates tests/golden/golden.json and golden_small.npz from the UNMODIFIED reference.

Run in the build container (where /root/reference exists and oracle/_ref/libpaces_ref.so has been built by
`make -C oracle ref`):  python tests/golden/make_golden.py
The fixtures are committed; the GPU box only reads them.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from oracle.pyoracle import ModelDef, fnv1a64, load_reference  # noqa: E402
from cases import CASES  # noqa: E402


def main():
    ref = load_reference()
    assert ref.impl == "reference"
    out = {}
    for name, case in CASES.items():
        m = ref.model(ModelDef(**case["model"]))
        run = m.run(**case["run"])
        rows, nnz, t, _ = run.info()
        w, c = run.state()
        rp, col, val = run.csr()
        rec = dict(layout=dict(sites=m.layout_sites, words=m.words, bits=m.total_bits, terms=m.n_terms),
                   init=dict(q_true=rows, nnz=nnz, table=fnv1a64(w), coeff=fnv1a64(c), col=fnv1a64(col), val=fnv1a64(val)),
                   snaps={})
        for s in range(1, case["steps"] + 1):
            d = run.step()
            if s in case["snaps"]:
                w, c = run.state()
                rp, col, val = run.csr()
                rec["snaps"][str(s)] = dict(diag=d, nnz=int(rp[-1]), table=fnv1a64(w), coeff=fnv1a64(c),
                                            row_ptr=fnv1a64(rp), col=fnv1a64(col), val=fnv1a64(val))
        ob = run.observe()
        ob["amp"] = [ob["amp"].real, ob["amp"].imag]
        ob["density"] = [float(x) for x in ob["density"]]
        rec["final_observe"] = ob
        out[name] = rec
        print(name, rec["snaps"][str(case["steps"])]["diag"]["q_true"], rec["snaps"][str(case["steps"])]["table"])

    with open(os.path.join(ROOT, "tests", "golden", "golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)

    # small full-array fixtures: apply_terms on a few keys, one grown space, one selection with ties
    small = {}
    m = ref.model(ModelDef(**CASES["disordered_4x3_d7"]["model"]))
    rng = np.random.RandomState(5)
    keys, amps, counts, srcs = [], [], [], []
    for _ in range(40):
        occ = np.concatenate([[rng.randint(12)], rng.randint(0, 7, 12)]).astype(np.uint32)
        k = m.pack(occ)
        nk, na = m.apply_terms(k)
        srcs.append(k); keys.append(nk); amps.append(na); counts.append(len(na))
    small["apply_src"] = np.array(srcs)
    small["apply_keys"] = np.concatenate(keys)
    small["apply_amps"] = np.concatenate(amps)
    small["apply_counts"] = np.array(counts)
    seeds = np.unique(np.array(srcs[:6]), axis=0)
    seeds = seeds[np.lexsort(seeds.T[::-1])]
    tw, rp, col, val = m.grow(seeds, 2)
    small.update(grow_seeds=seeds, grow_table=tw, grow_row_ptr=rp, grow_col=col, grow_val=val)
    # selection with a 4-way tie at the cutoff (test_engine.cpp:126-160 pattern)
    m2 = ref.model(ModelDef(kind=1, extents=(3,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(0.5,), d_pho=2))
    occs = [(0, 0, 0, 0), (0, 1, 0, 0), (1, 0, 0, 0), (1, 0, 1, 0), (2, 0, 0, 0), (2, 0, 0, 1), (2, 1, 1, 1)]
    words = np.array([m2.pack(o) for o in occs])
    order = np.lexsort(words.T[::-1]); words = words[order]
    coeff = np.array([0.9, 0.3, 0.3j, -0.3, 0.3, 0.1, 0.0], dtype=np.complex128)
    sel = {str(seed): m2.truncate_select(words, coeff, 3, seed) for seed in range(16)}
    small["sel_words"] = words
    small["sel_coeff"] = coeff
    for k, v in sel.items():
        small["sel_kept_" + k] = v
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "golden_small.npz"), **small)
    print("wrote golden fixtures")


if __name__ == "__main__":
    main()
