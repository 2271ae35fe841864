"""Run one hot-path call back to back for a few seconds and sample SM clock / power / throttle
reasons with nvidia-smi meanwhile (is the kernel power-capped?).

    python tools/power_probe.py fwd|bwd|fwd128|sq [seconds]
"""
import os, subprocess, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_05682_b200 import api

what = sys.argv[1]
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 4.0
d = 128 if what == "fwd128" else 64
q = torch.empty((1, 16384, 16, d), dtype=torch.bfloat16, device="cuda")
k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
for t, tid in ((q, 1), (k, 2), (v, 3), (do, 4)):
    api.mea_fill_synthetic(t, 0, tid)
out, lse = api.mea_attention_fwd(q, k, v, want_lse=True)
fn = {"fwd": lambda: api.mea_attention_fwd(q, k, v, out=out, lse=lse),
      "fwd128": lambda: api.mea_attention_fwd(q, k, v, out=out, lse=lse),
      "bwd": lambda: api.mea_attention_bwd(q, k, v, out, do, lse=lse)}[what]
samples = []
stop = False


def sampler():
    while not stop:
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                            "--format=csv,noheader,nounits", "-i", "0"], capture_output=True, text=True).stdout
        samples.append(r.strip())
        time.sleep(0.1)


fn(); torch.cuda.synchronize()
th = threading.Thread(target=sampler); th.start()
t0 = time.time(); n = 0
e0 = torch.cuda.Event(True); e0.record()
while time.time() - t0 < secs:
    for _ in range(20):
        fn()
    n += 20
    torch.cuda.synchronize()
e1 = torch.cuda.Event(True); e1.record(); torch.cuda.synchronize()
stop = True; th.join()
print(f"{what}: {n} calls, {e0.elapsed_time(e1) / n:.3f} ms per call")
for s in samples[::max(1, len(samples) // 12)]:
    print("  sm_mhz, W, reasons:", s)
