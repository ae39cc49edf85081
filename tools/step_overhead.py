"""Bench-step overhead experiment: library stream vs torch stream, with/without the L2 flush."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
g = load_config("c5")
stream = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def run(label, use_stream, do_flush, steps=8):
    for _ in range(2):
        vc.solve_pvc(g, 482, strategy="gpu", stream=stream.cuda_stream if use_stream else None)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dev = []
    t0 = time.perf_counter()
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for _ in range(steps):
            r = vc.solve_pvc(g, 482, strategy="gpu", stream=stream.cuda_stream if use_stream else None)
            dev.append(r["device_ms"])
            if do_flush:
                flush.zero_()
        ev1.record(stream)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print(f"{label}: event {ev0.elapsed_time(ev1)/steps:.2f} ms/step, host {t*1e3/steps:.2f} ms/step, device {sum(dev)/steps:.2f}", flush=True)
run("lib stream, no flush", False, False)
run("torch stream, no flush", True, False)
run("torch stream, flush", True, True)
run("lib stream, flush", False, True)
import bench
cs = bench.ClockSampler(0); cs.start(); time.sleep(0.5)
run("lib stream, flush, nvidia-smi sampler running", False, True, steps=20)
print(cs.stop())
cs = bench.ClockSampler(0); cs.start(); time.sleep(0.5)
run("torch stream, flush, nvidia-smi sampler running", True, True, steps=20)
print(cs.stop())
import pynvml, threading
pynvml.nvmlInit(); hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
stop = False; samples = []
def loop():
    while not stop:
        samples.append((pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(hnd)))
        time.sleep(0.05)
th = threading.Thread(target=loop, daemon=True); th.start(); time.sleep(0.2)
run("lib stream, flush, pynvml 50ms sampler", False, True, steps=20)
stop = True; th.join(); print(len(samples), samples[-3:])
