"""CPU ORACLE — test infrastructure only (never imported by the product path).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package, and only as the checker / the CPU
baseline. The executor (paper_2405_01248_b200) never calls into it.

Contents
  nets.py       fp32 PyTorch (CPU) restatement of every model component the
                executor runs, over the same named parameters (plain F.* ops).
  train_step.py the sequential, non-pipelined diffusion training step with
                frozen encoders, self-conditioning and AdamW: the numerical
                oracle of the pipelined step (cross-iteration equivalence,
                PAPER.md:294-300; self-conditioning).

Schedule/partition oracle: the reference planner itself (`pipefill`,
/root/reference/pkg/src here, baseline/_ref on the GPU box), pinned by
tests/golden/planner_cases.json.

Parity status: the schedule side is pinned bit-exactly by the reference's own
outputs (golden fixtures + live comparison). The numerics side has NO
reference implementation (the paper's back-end is not in /root/reference,
SURVEY.md §8c): this restatement is written from the paper's training
semantics and standard PyTorch ops — numerics parity is "unpinned" by the
reference and is stated as such in DESIGN.md.
"""
