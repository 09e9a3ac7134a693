"""One tiny pipelined training iteration of config c1 on cuda:0, checked against the
CPU oracle (used here only as the checker). Raises on any mismatch or if the native
library is missing."""

from __future__ import annotations


def run_smoke():
    import torch

    from . import diffusion, engine, nn, telemetry

    if not torch.cuda.is_available():
        raise RuntimeError("smoke() needs a CUDA device")
    torch.cuda.set_device(0)
    telemetry.reset()
    tr = engine.Trainer.create("c1", world=1, rank=0, S=1, M=2, D=1, world_batch=4, device="cuda:0")
    loss = tr.step(has_next=False).item()
    torch.cuda.synchronize()
    from oracle import train_step

    m = tr.model
    params = {c.name: nn.init_state(c.store.param_specs(), 0)
              for c in [m.backbone] + [f.component for f in m.frozen]}
    sab, s1m = diffusion.noise_schedule()
    ref, _, _ = train_step.train("c1", params, [diffusion.make_batch(tr.data_spec, 0)], sab, s1m)
    if abs(loss - ref[0]) > 1e-4 * abs(ref[0]) + 1e-6:
        raise AssertionError(f"smoke: loss {loss} != oracle {ref[0]}")
    n = telemetry.total_launches()
    if n == 0:
        raise AssertionError("smoke: no libdpipe kernels launched")
    print(f"smoke ok: c1 loss {loss:.6f} (oracle {ref[0]:.6f}), {n} libdpipe kernel launches")
