"""Shared-memory bank model of the brick query's corner loads (K1).

A warp's 32 lanes each evaluate one point of a brick (Morton-ordered within
the brick, ~0.5 points per cell) and read the K-float blocks of its cell's 8
corners from a tile with row stride TROWF and plane stride PLANE floats, with
LDW-float loads. Prints the modelled wavefronts per warp-wide load
instruction (a phase of 32/LDW lanes costs the max over banks of distinct
addresses; identical addresses broadcast).

    python tools/bank_model.py [K] [TROWF] [PLANE] [LDW]
"""
import sys

import numpy as np


def spread(x):
    r = 0
    for b in range(3):
        r |= ((x >> b) & 1) << (3 * b)
    return r


def morton(cx, cy, cz):
    return spread(cx) | (spread(cy) << 1) | (spread(cz) << 2)


def wavefronts(K, trowf, plane, ldw=2, trials=30, npts=256, seed=0):
    rng = np.random.default_rng(seed)
    tot = cnt = 0
    per = 32 // ldw
    for _ in range(trials):
        c = rng.integers(0, 8, (npts, 3))
        c = c[np.argsort([morton(*x) for x in c], kind="stable")]
        for w in range(npts // 32):
            cc = c[w * 32:(w + 1) * 32]
            for corner in range(8):
                v = cc + np.array([corner & 1, (corner >> 1) & 1, (corner >> 2) & 1])
                base = v[:, 0] * K + v[:, 1] * trowf + v[:, 2] * plane
                for q in range(K // ldw):
                    word = base + ldw * q
                    for ph in range(ldw):
                        addrs = np.unique(word[ph * per:(ph + 1) * per])
                        banks = np.concatenate([(addrs + k) % 32 for k in range(ldw)])
                        tot += np.bincount(banks, minlength=32).max()
                        cnt += 1
    return tot / cnt * ldw


if __name__ == "__main__":
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    tr = int(sys.argv[2]) if len(sys.argv) > 2 else 104
    pl = int(sys.argv[3]) if len(sys.argv) > 3 else 9 * tr
    ldw = int(sys.argv[4]) if len(sys.argv) > 4 else (2 if K % 4 else 4)
    print(f"K={K} TROWF={tr} PLANE={pl} LDW={ldw}: {wavefronts(K, tr, pl, ldw):.2f} wavefronts per load")
