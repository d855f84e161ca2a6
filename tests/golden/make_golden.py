"""Generates tests/golden/*.npz from the UNMODIFIED reference library (oracle/_ref,
built from /root/reference by oracle/Makefile). Run in the build container:

    python tests/golden/make_golden.py

The fixtures are small and committed, so parity tests on the GPU box (where
/root/reference does not exist) still compare against reference outputs."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Reference, build  # noqa: E402


def main():
    build()
    ref = Reference()
    F, H, W, C, groups, nl, ng, seed, wseed, t = 16, 4, 4, 32, 4, 8, 4, 0, 1, 900.0
    x = ref.fill_seeded(F * H * W * C, seed).reshape(F, H, W, C)
    bp = ref.build_block(C, 3, groups, wseed)
    y = ref.block_forward(x, 3, groups, wseed, t, n_local=nl, n_global=ng)
    y2, _ = ref.block_forward(x, 3, groups, wseed, t, n_local=nl, n_global=ng, workers=2,
                              traffic=True)
    np.savez_compressed(os.path.join(HERE, "block_small.npz"), x=x, y=y, y_workers2=y2, C=C,
                        groups=groups, n_local=nl, n_global=ng, weight_seed=wseed, t=t,
                        stub_a=bp.stub_a, conv_w=bp.conv_w, wq=bp.wq, wo=bp.wo)
    # token sets / plans / traffic (integer goldens)
    sets = {f"gset_{f}_{n}": np.array(ref.build_global_index_set(f, n), np.uint32)
            for f, n in [(24, 16), (48, 16), (192, 16), (2300, 16), (2304, 16), (100, 64)]}
    traffic = np.array([ref.predict_sync_traffic(f, n, h, g, w, 1 << 20)
                        for f, n, h, g in [(48, 2, 8, 16), (96, 4, 8, 16), (192, 8, 8, 16),
                                           (2304, 8, 8, 16)] for w in range(n)], np.uint64)
    np.savez_compressed(os.path.join(HERE, "index_sets.npz"), traffic=traffic, **sets)
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
