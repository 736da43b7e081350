#!/usr/bin/env python
"""Sweep measurement of heavy sizes, twice: policy times must agree between passes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200 import sweep

    sizes = [sk.ProblemSize(8192, 14336, 4096), sk.ProblemSize(4096, 14336, 4096), sk.ProblemSize(8192, 4096, 4096),
             sk.ProblemSize(2048, 14336, 4096)]
    tile = sk.TileShape(256, 256, 128)
    for rep in range(2):
        for rec in sweep.tune_sizes(sizes, tile):
            print(rep, f"{rec.size.m}x{rec.size.n}x{rec.size.k}", " ".join(f"{p.label}:{e.makespan:.0f}" for p, e in rec.costs),
                  "->", rec.winner.label, flush=True)


if __name__ == "__main__":
    main()
