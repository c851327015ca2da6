import sys, os, torch, json
sys.path.insert(0, os.getcwd())
import synth, paper_1807_07433_b200 as rsr
cfg = synth.get_config("c5"); B = 8
left, right, ab = synth.make_batch(cfg, list(range(B)))
L = torch.from_numpy(left).cuda(); R = torch.from_numpy(right).cuda(); A = torch.from_numpy(ab).cuda()
pipe = rsr.StereoPipeline(B, cfg.height, cfg.width, rsr.StereoParams.from_config(cfg))
p = pipe.p; main = torch.cuda.current_stream(); side = torch.cuda.Stream()
def step(conc):
    rsr.rsr_warp(R, A, pipe.warped, pipe.valid, pipe.shift)
    rsr.rsr_cost_volume(L, pipe.warped, pipe.valid, p.rho_block, p.d_lo, p.d_hi, vol_ref=pipe.vol_ref,
                        vol_tar=pipe.vol_tar, nan_ref=pipe.nan_ref, nan_tar=pipe.nan_tar, workspace=pipe.workspace)
    if conc:
        e = torch.cuda.Event(); e.record(main); side.wait_event(e)
        with torch.cuda.stream(side):
            rsr.rsr_aggregate(pipe.vol_tar, pipe.warped, p.rho_agg, p.gamma_d, p.gamma_r, pipe.nan_tar, pipe.agg_tar)
        rsr.rsr_aggregate(pipe.vol_ref, L, p.rho_agg, p.gamma_d, p.gamma_r, pipe.nan_ref, pipe.agg_ref)
        e2 = torch.cuda.Event(); e2.record(side); main.wait_event(e2)
    else:
        rsr.rsr_aggregate(pipe.vol_ref, L, p.rho_agg, p.gamma_d, p.gamma_r, pipe.nan_ref, pipe.agg_ref)
        rsr.rsr_aggregate(pipe.vol_tar, pipe.warped, p.rho_agg, p.gamma_d, p.gamma_r, pipe.nan_tar, pipe.agg_tar)
    rsr.rsr_disparity(pipe.agg_ref, pipe.agg_tar, pipe.shift, p.d_lo, p.d_hi, p.lrc_tol, True, pipe.disparity)
    rsr.rsr_reconstruct(pipe.disparity, p.focal, p.baseline, d_min=p.d_min, xyz=pipe.xyz)
for conc in (False, True, False, True):
    for _ in range(3): step(conc)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): step(conc)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(json.dumps({"concurrent_k3": conc, "ms_per_step": ms, "fps": B / ms * 1e3}))
