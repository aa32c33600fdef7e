"""Golden fixtures for the GPU quantizer, written by the REAL reference's
fitting API (bcq.py greedy_init / ls_update_scales / bs_recalibrate_codes /
alternate_fit, progressive.py build_multiprecision). Build container only:

    python tests/golden/make_golden_quant.py

Outputs tests/golden/quant_*.npz: the input matrix, the reference's packed
words, f32 scales / offsets and the alternate_fit error trace.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from make_golden import _import_reference  # noqa: E402

CASES = [
    # name, rows, cols, group, mode, q / (p_lo, p_hi), cycles, kind
    ("greedy_sym", 48, 256, 128, "symmetric", 3, 0, "greedy"),
    ("greedy_asym_g40", 20, 120, 40, "asymmetric", 3, 0, "greedy"),
    ("alt_sym", 32, 256, 128, "symmetric", 3, 3, "alternate"),
    ("alt_asym_g64", 24, 256, 64, "asymmetric", 2, 3, "alternate"),
    ("multi_sym", 64, 512, 128, "symmetric", (2, 4), 2, "multi"),
    ("multi_asym_g32", 32, 128, 32, "asymmetric", (1, 3), 2, "multi"),
    ("multi_sym_c0", 16, 256, 128, "symmetric", (2, 3), 0, "multi"),
]


def main():
    A = _import_reference()
    from anybcq.bcq import alternate_fit, bs_recalibrate_codes, greedy_init, ls_update_scales
    from anybcq.progressive import build_multiprecision

    for ci, (name, rows, cols, g, mode, q, cycles, kind) in enumerate(CASES):
        w = A.random_gaussian(rows, cols, seed=40 + ci)
        cfg = A.QuantConfig(group_size=g, mode=mode, cycles=cycles)
        out = {"w": w, "group_size": g, "asym": int(mode == "asymmetric"), "cycles": cycles}
        if kind == "greedy":
            qm = greedy_init(w, q, cfg)
            out.update(words=qm.bitplanes.words, alpha=qm.scales.alpha, q=q)
            if qm.scales.offset is not None:
                out["offset"] = qm.scales.offset
            st = ls_update_scales(w, qm)
            out["ls_alpha"] = st.alpha
            if st.offset is not None:
                out["ls_offset"] = st.offset
            out["bs_words"] = bs_recalibrate_codes(w, st).words
        elif kind == "alternate":
            trace = []
            qm = alternate_fit(w, q, cfg, trace=trace)
            out.update(words=qm.bitplanes.words, alpha=qm.scales.alpha, q=q, trace=np.asarray(trace))
            if qm.scales.offset is not None:
                out["offset"] = qm.scales.offset
        else:
            m = build_multiprecision(w, q[0], q[1], cfg)
            out.update(words=m.bitplanes.words, p_lo=q[0], p_hi=q[1])
            for p in m.precisions:
                out[f"alpha_{p}"] = m.scale_sets[p].alpha
                if m.scale_sets[p].offset is not None:
                    out[f"offset_{p}"] = m.scale_sets[p].offset
        np.savez_compressed(HERE / f"quant_{name}.npz", **out)
        print("wrote", name)


if __name__ == "__main__":
    main()
