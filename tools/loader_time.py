#!/usr/bin/env python3
"""MFW1 blob -> device-resident compute layout, GPT-2-medium shape (c2):
host path (load_weights + numpy transposes + per-array uploads) vs
load_weights_device (one pinned H2D + native transpose/cast)."""
import os, sys, tempfile, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2104_12470_b200 as eet  # noqa: E402
from paper_2104_12470_b200.weights import DeviceModel  # noqa: E402
from paper_2104_12470_b200.core import dtype_code  # noqa: E402


def main():
    cfg = eet.ModelConfig(16, 1024, 24, 16, 512, 1024, datatype_label="fp16")
    w = eet.random_weights(cfg, 50257, seed=0)
    path = os.path.join(tempfile.mkdtemp(), "gpt2m.mfw1")
    eet.save_weights(w, path)
    dt = dtype_code("fp16")
    torch.cuda.synchronize()
    for name, fn in [("host  ", eet.load_weights), ("device", eet.load_weights_device),
                     ("host  ", eet.load_weights), ("device", eet.load_weights_device)]:
        t0 = time.perf_counter()
        wl = fn(path)
        DeviceModel.of(wl, dt)
        torch.cuda.synchronize()
        print(f"{name} blob {os.path.getsize(path) / 1e9:.2f} GB -> device fp16 layout: "
              f"{time.perf_counter() - t0:.2f} s", flush=True)
        del wl
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
