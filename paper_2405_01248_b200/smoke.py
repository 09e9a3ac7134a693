"""Smoke test on cuda:0, checked against the CPU oracle (used here only as the checker).
Raises on any mismatch or if the native library is missing.

1. config c2 with a 2-layer text encoder (bf16: the tcgen05/TMEM/TMA GEMM, convolution and fused
   flash-attention kernels that carry the benchmark), one iteration with cross-iteration filling
   and the overlapped optimizer, loss rtol 2e-2 (BASELINE.json north_star bf16 tolerance);
2. config c1 (tiny DiT, fp32: the SIMT GEMM path), one pipelined iteration, loss rtol 1e-4."""

from __future__ import annotations


def run_smoke():
    import torch

    from . import diffusion, engine, nn, telemetry

    if not torch.cuda.is_available():
        raise RuntimeError("smoke() needs a CUDA device")
    torch.cuda.set_device(0)
    from oracle import train_step

    sab, s1m = diffusion.noise_schedule()
    msgs = []
    # c2 first: its bf16 tensor-core kernels lead the launch list a profiler records
    for cfg, kw, tol, small in (("c2", dict(clip_layers=2), 2e-2, True), ("c1", {}, 1e-4, False)):
        telemetry.reset()
        tr = engine.Trainer.create(cfg, world=1, rank=0, S=1, M=2 if cfg == "c1" else 1, D=1,
                                   world_batch=4 if cfg == "c1" else 2, device="cuda:0", small=small)
        loss = tr.step(has_next=cfg != "c1").item()
        torch.cuda.synchronize()
        n = telemetry.total_launches()
        fams = dict(telemetry.launches)
        m = tr.model
        params = {c.name: nn.init_state(c.store.param_specs(), 0)
                  for c in [m.backbone] + [f.component for f in m.frozen]}
        ref, _, _ = train_step.train(cfg, params, [diffusion.make_batch(tr.data_spec, 0)], sab, s1m, **kw)
        if abs(loss - ref[0]) > tol * abs(ref[0]) + 1e-6:
            raise AssertionError(f"smoke {cfg}: loss {loss} != oracle {ref[0]} (rtol {tol})")
        if n == 0:
            raise AssertionError(f"smoke {cfg}: no libdpipe kernels launched")
        if cfg == "c2" and not all(fams.get(k) for k in ("dp_gemm", "dp_conv_fwd", "dp_flash_attn_fwd")):
            raise AssertionError(f"smoke c2: bf16 tensor-core kernels missing from the launches {fams}")
        msgs.append(f"{cfg} loss {loss:.6f} (oracle {ref[0]:.6f}, {n} libdpipe launches)")
        del tr, m
        torch.cuda.empty_cache()
    print("smoke ok: " + "; ".join(msgs))
