"""Tuning sweep (GPU): time one layout over configs x plan knobs.

  python tools/sweep.py --configs d16_1e6,lowd1_1e7 --layout tiled --tpi 1,2 --ns 3,6 --nbuf 1,2 --tile -1

Knobs are the plan builder's tuning hooks (env P2P_TPI / P2P_NS / P2P_NBUF,
read at plan build) and the descriptor's tile_log2.  Prints one line per
variant: median kernel time (CUDA events, L2 flushed between reps), Gpair/s,
fraction of the MUFU roofline and algorithmic GB/s."""
import argparse
import itertools
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_01596_b200 import p2p  # noqa: E402
from paper_2403_01596_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="d16_1e6,d64_1e6,lowd1_1e7")
    ap.add_argument("--layout", default="tiled")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--tpi", default="1,2")
    ap.add_argument("--ns", default="3,6")
    ap.add_argument("--nbuf", default="1,2")
    ap.add_argument("--tile", default="-1")
    ap.add_argument("--nt", default="128")
    ap.add_argument("--pad", default="1")
    ap.add_argument("--lpt", default="", help="P2P_LPT values (comma list; empty = plan default)")
    ap.add_argument("--tail", default="", help="tail splitting as TILES:PARTS (comma list; empty = default)")
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--json", default="")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    peak = 16 * 148 * 1.965e9
    rows = []
    for name in args.configs.split(","):
        cfg = W.CONFIGS[name]
        src, tgt, q = W.make_problem(cfg)
        for tpi, ns, nbuf, tile, nt, pad, lpt, tail in itertools.product(
                args.tpi.split(","), args.ns.split(","), args.nbuf.split(","), args.tile.split(","),
                args.nt.split(","), args.pad.split(","), args.lpt.split(","), args.tail.split(",")):
            for key, val in (("P2P_LPT", lpt), ("P2P_TAIL_TILES", tail.split(":")[0] if tail else ""),
                             ("P2P_TAIL_PARTS", tail.split(":")[1] if tail else "")):
                if val:
                    os.environ[key] = val
                else:
                    os.environ.pop(key, None)
            if tpi == "2" and pad == "0":
                continue
            os.environ["P2P_TPI"], os.environ["P2P_NS"], os.environ["P2P_NBUF"] = tpi, ns, nbuf
            os.environ["P2P_NT"], os.environ["P2P_PAD"] = nt, pad
            try:
                pl = p2p.Plan(src, tgt, level=cfg.level, layout=args.layout, precision=args.precision, device=0,
                              tile_log2=int(tile))
            except p2p.P2PError as e:
                print(name, tpi, ns, nbuf, tile, "plan failed:", e)
                continue
            qd = torch.as_tensor(q[pl.export("src_perm")], dtype=pl.torch_dtype, device=dev)
            out = torch.empty(pl.info["n_tgt_local"], dtype=pl.torch_dtype, device=dev)
            for _ in range(3):
                pl.apply(qd, out)
            ts = []
            for _ in range(args.reps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                pl.apply(qd, out)
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
            ms = float(np.median(ts))
            i = pl.info
            row = dict(config=name, tpi=tpi, ns=ns, nbuf=nbuf, nt=nt, pad=pad, lpt=lpt, tail=tail,
                       tile=i["tile_log2"], smem=i["smem_bytes"],
                       us=ms * 1e3, gpair=i["pairs"] / ms / 1e6, frac=i["pairs"] / (ms * 1e-3) / peak,
                       alg_gbs=i["alg_bytes_kernel"] / ms / 1e6, lay_gbs=i["layout_bytes_apply"] / ms / 1e6)
            rows.append(row)
            print(f"{name:12s} tpi {tpi} ns {ns} nbuf {nbuf} nt {nt} pad {pad} lpt {lpt or '-'} tail {tail or '-'} "
                  f"k {i['tile_log2']} smem {i['smem_bytes']:6d} "
                  f"{ms * 1e3:8.1f} us {row['gpair']:8.1f} Gpair/s mufu {row['frac']:.3f} alg {row['alg_gbs']:6.0f} layout {row['lay_gbs']:6.0f} GB/s",
                  flush=True)
            pl.close()
    if args.json:
        json.dump(rows, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
