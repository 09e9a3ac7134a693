"""Does clock sampling perturb the step? c2 N=1 step time with no sampler / nvidia-smi -lms 200 /
in-process NVML thread (diagnostics for bench.py's Clocks)."""
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import engine  # noqa: E402

tr = engine.Trainer.create("c2", world=1, rank=0, S=1, M=1, D=1, world_batch=32)
tr.prefetch(80)
for _ in range(3):
    tr.step()


def run(label):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        tr.step()
    b.record()
    torch.cuda.synchronize()
    print(label, "ms/step", round(a.elapsed_time(b) / 10, 2), flush=True)


run("none")
p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,clocks_event_reasons.active",
                      "--format=csv,noheader", "-lms", "200"], stdout=subprocess.DEVNULL)
time.sleep(0.5)
run("nvidia-smi-200ms")
p.terminate()
p.wait()
run("none")
import pynvml  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
stop = False
samples = []


def loop():
    while not stop:
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.2)


t = threading.Thread(target=loop)
t.start()
run("nvml-thread-200ms")
stop = True
t.join()
print("nvml samples", samples[:3])
run("none")
