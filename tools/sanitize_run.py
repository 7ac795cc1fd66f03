"""Small invocations of every kernel of libstyleblit for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): run as
    compute-sanitizer --tool TOOL --error-exitcode 9 python tools/sanitize_run.py [--quick]
on a GPU box (tools/sanitize.sh).  Covers configs 1 and 2 (r = 0 and r = 2), L = 3 / 5 / 12,
with and without the strided exemplar copy, ragged widths, row strips, the vote alone at
r = 1..7, the LUT builders and the host-buffer pipeline.  Outputs are only synchronised, not
checked (tests/ does parity); the sanitizer's verdict is the result."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1807_03249_b200 as sb  # noqa: E402
import synth  # noqa: E402


def main() -> None:
    quick = "--quick" in sys.argv
    dev = torch.device("cuda:0")
    runs = []
    for cid in (1, 2):
        cfg, cs, gs, gt = synth.config(cid)
        if quick and cid == 2:  # racecheck is slow: a 256-row strip of config 2 keeps every kernel path
            gt = gt[:256].contiguous()
        cs, gs, gt = cs.to(dev), gs.to(dev), gt.to(dev)
        lut = sb.build_lut(gs)
        ex = sb.prepare_exemplar(cs, gs)
        for L in (3, 5, 12):
            for r in (0, 2):
                for use_ex in (False, True):
                    prm = sb.Params(threshold=cfg["t"], levels=L, blend_radius=r, guide_channels=cfg["C"],
                                    seed=cfg["seed"], exemplar=ex if use_ex else None)
                    sb.stylize(prm, cs, gs, lut, gt)
                    runs.append((cid, L, r, use_ex))
        # ragged width (wt % 4 != 0) and a row strip
        gtr = gt[:, : gt.shape[1] - 3].contiguous()
        for r in (0, 2):
            sb.stylize(sb.Params(threshold=cfg["t"], levels=cfg["L"], blend_radius=r, guide_channels=cfg["C"]),
                       cs, gs, lut, gtr)
            sb.stylize(sb.Params(threshold=cfg["t"], levels=cfg["L"], blend_radius=r, guide_channels=cfg["C"],
                                 row_begin=5, row_end=gt.shape[0] - 7, exemplar=ex), cs, gs, lut, gt)
        # the level map, weights + label (EXT), the 3-channel table
        sb.stylize(sb.Params(threshold=cfg["t"], levels=cfg["L"], guide_channels=cfg["C"], weights=(1, 2, 3, 0),
                             label_channel=3), cs, gs, lut, gt)
        if cid == 1 or not quick:
            lut3 = sb.build_lut3(gs)
            sb.stylize(sb.Params(threshold=cfg["t"], levels=cfg["L"], guide_channels=cfg["C"], lut_rgb=True,
                                 exemplar=ex), cs, gs, lut3, gt)
            del lut3
        # the vote alone, r = 1..7
        _, coords, _ = sb.stylize(sb.Params(threshold=cfg["t"], levels=cfg["L"], guide_channels=cfg["C"]),
                                  cs, gs, lut, gt)
        for r in range(1, 8):
            sb.vote(coords, cs, r)
            sb.vote(coords, cs, r, exemplar=ex)
        # batch with per-frame seeds, and the host pipeline
        gtb = gt.unsqueeze(0).repeat(3, 1, 1, 1).contiguous()
        sb.stylize_batch(sb.Params(threshold=cfg["t"], levels=cfg["L"], guide_channels=cfg["C"], exemplar=ex),
                         cs, gs, lut, gtb, frame_seeds=[1, 2, 3])
        gth = gtb.cpu().pin_memory()
        cth = torch.empty_like(gth).pin_memory()
        sb.stylize_batch_host(sb.Params(threshold=cfg["t"], levels=cfg["L"], guide_channels=cfg["C"], blend_radius=2,
                                        exemplar=ex), cs, gs, lut, gth, cth, depth=2)
        torch.cuda.synchronize()
        print(f"config {cid}: ok ({len(runs)} stylize variants so far)", flush=True)
    print("sanitize_run done", flush=True)


if __name__ == "__main__":
    main()
