"""Multi-rank control plane on CPU (gloo, world 2 and 4): the pipelined executor
(stage partition, live-set P2P in both directions, self-conditioning feedback,
cross-iteration bubble fills with partial batches and frozen-activation transfers,
per-stage gradient allreduce across replicas and groups, flat AdamW) must produce the
same losses and parameters as the single-rank sequential run of the same model.

The compute is a tiny torch-op model (tests/cpu_pipeline_model.py) — test-only; on
B200 the same executor runs the libdpipe components.
"""

import os
import socket
import sys

import pytest
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

ITERS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _make(world, rank, S, M, D, selfcond, wb, deps=False, two=False, program_file=None):
    import cpu_pipeline_model as cm
    from paper_2405_01248_b200 import engine
    from paper_2405_01248_b200.diffusion import DataSpec

    model = cm.build(selfcond, deps=deps, two=two)
    ds = DataSpec(7, wb, cm.IMG, cm.LAT, cm.ZC, cm.TL, cm.VOCAB, 1000, 0.5 if selfcond else 0.0)
    cfg = engine.ConfigSpec("toy", torch.float32, cm.IMG, cm.LAT, cm.TL, cm.VOCAB, ds.selfcond_p, 7)
    return engine.Trainer.from_model(model, cfg, ds, world=world, rank=rank, S=S, M=M, D=D, device="cpu",
                                     program_file=program_file)


def _worker(rank, world, S, M, D, selfcond, wb, port, outdir, deps=False, two=False, from_file=False):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    tr = _make(world, rank, S, M, D, selfcond, wb, deps, two)
    if from_file:
        # ship the plan as per-rank program files (rank 0 writes them), then run from the files
        import dataclasses

        pdir = os.path.join(outdir, "programs")
        if rank == 0:
            tr.save_programs(pdir)
        dist.barrier()
        planned = tr
        tr = _make(world, rank, S, M, D, selfcond, wb, deps, two,
                   program_file=os.path.join(pdir, f"rank{rank}.json"))
        for k in (False, True):
            assert dataclasses.asdict(tr.ex.programs[k]) == dataclasses.asdict(planned.ex.programs[k])
        assert dataclasses.asdict(tr.ex.warm_program) == dataclasses.asdict(planned.ex.warm_program)
        del planned
    losses = []
    for i in range(ITERS):
        dist.barrier()
        tr.step(has_next=i < ITERS - 1, trace=i == ITERS - 2)
        losses.append(tr.ex.total_loss().item())
        if i == ITERS - 2:
            sched, bubbles, ratio = tr.measured()
            mine = tr.ex.measured_tasks()
    prog = tr.ex.programs[True]
    params = []
    for pi, rng in enumerate(tr.ex.param_ranges):
        if rng is not None:
            bi = prog.pipes[pi].backbone
            lo, hi = rng
            params.append((bi, lo, hi, tr.model.backbones[bi].store.flat.detach()[lo:hi].clone()))
    torch.save(dict(losses=losses, params=params, npipes=len(prog.pipes),
                    transfers=len(prog.transfers), fills=sum(len(f) for f in prog.fills),
                    tail=len(prog.tail), ratio=ratio, ntasks=len(sched.tasks), mine=mine,
                    instrs=[i[0] for i in tr.ex.prog.device_program(tr.ex.dev).instrs],
                    makespan=sched.makespan),
               os.path.join(outdir, f"r{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def _reference(selfcond, wb, deps=False, two=False):
    tr = _make(1, 0, 1, 1, 1, selfcond, wb, deps, two)
    losses = []
    for i in range(ITERS):
        tr.step(has_next=i < ITERS - 1)
        losses.append(tr.ex.total_loss().item())
    return losses, [b.store.flat.detach().clone() for b in tr.model.backbones]


@pytest.mark.parametrize("world,S,M,D,selfcond,deps,two", [
    (2, 2, 4, 2, False, False, False),
    (2, 2, 4, 2, True, False, False),
    (4, 2, 2, 2, True, False, False),     # 2 pipeline groups (DP across groups)
    (4, 2, 4, 4, False, False, False),    # 2 replicas per stage (DP inside a stage)
    (2, 2, 4, 2, False, True, False),     # frozen component depending on two others (ControlNet-like)
    (2, 2, 4, 2, False, False, True),     # two backbones, bidirectional pipelines
    (2, 2, 4, 2, True, False, True),      # bidirectional + self-conditioning feedback per pipe
])
def test_pipelined_equals_sequential(tmp_path, world, S, M, D, selfcond, deps, two, from_file=False):
    import torch.multiprocessing as mp

    wb = 16 * (world // D)
    mp.spawn(_worker, args=(world, S, M, D, selfcond, wb, _free_port(), str(tmp_path), deps, two, from_file),
             nprocs=world, join=True)
    ref_losses, ref_flats = _reference(selfcond, wb, deps, two)
    outs = [torch.load(os.path.join(tmp_path, f"r{r}.pt"), weights_only=False) for r in range(world)]
    covered = [torch.zeros(f.numel(), dtype=torch.bool) for f in ref_flats]
    for o in outs:
        assert o["npipes"] == (2 if two else 1)
        for a, b in zip(o["losses"], ref_losses):
            assert abs(a - b) <= 1e-5 * abs(b) + 1e-7, (o["losses"], ref_losses)
        for bi, lo, hi, p in o["params"]:
            assert torch.allclose(p, ref_flats[bi][lo:hi], rtol=1e-5, atol=1e-6)
            covered[bi][lo:hi] = True
    assert all(c.all() for c in covered)
    # measured schedule of a traced iteration: one task per executed instruction, compute
    # tasks in program order, a bubble ratio in [0, 1) from the planner's own definitions
    for o in outs:
        kinds = [t.kind for t in o["mine"]]
        assert len(kinds) == len(o["instrs"]), (kinds, o["instrs"])
        comp = [t for t in o["mine"] if t.kind in ("fwd", "bwd", "fwd_sc")]
        assert all(a.end <= b.start + 1e-9 for a, b in zip(comp, comp[1:]))
        assert 0.0 <= o["ratio"] < 1.0 and o["makespan"] > 0
        assert o["ntasks"] == sum(len(x["mine"]) for x in outs) // (world // D)
    # the fill plan actually exercised bubbles (and, with several devices, frozen transfers)
    # (bidirectional plans leave bubbles too short to fill at this toy size)
    assert two or any(o["fills"] > 0 for o in outs)


def test_pipelined_from_shipped_program_files(tmp_path):
    """PAPER.md:266 instruction generation as a standalone artefact: the job runs from per-rank
    program files (adapter.save_rank_programs / load_rank_program, format dpipe-program/v1) that
    round-trip the planned programs exactly, with the sequential run's losses and parameters
    (2 pipeline groups x 2 stages, self-conditioning, fills with frozen transfers)."""
    test_pipelined_equals_sequential(tmp_path, 4, 2, 2, 2, True, False, False, from_file=True)
