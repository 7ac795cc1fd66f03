import torch, synth, paper_1807_03249_b200 as sb
cfg = synth.CONFIGS[5]
cs, gs = [t.cuda() for t in synth.exemplar(cfg, device="cuda")]
gt = synth.heightfield_normals(3840, 2160, seed=5, frame=0, device="cuda").unsqueeze(0)
prm = sb.Params(threshold=cfg["t"], levels=5, flags=sb.SB_NO_COLOR)
lut = sb.build_lut(gs)
_, co, _ = sb.stylize_batch(prm, cs, gs, lut, gt, want_level=False)
ct = sb.vote(co, cs, 2)
torch.cuda.synchronize()
print("ok")
