"""Cross-process row bands (BASELINE config 5): one process per
band, launched by torchrun. Rank 0 encodes the frame into a banded bitstream
(in-process group on its own GPU), every rank decodes its band through its
own handle with the halo K/V exchanged by P2P stores + device mailbox flags,
and rank 0 checks the assembled latents bit-exact and prints one JSON line.

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
      --master-port P tools/band_ranks.py [--preset paper --height 136 --width 240]

--same-device puts every rank on cuda:0 (the 1-GPU CI case: contexts
time-slice, so it checks correctness, not speed)."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2605_20977_b200 import dist as pdist  # noqa: E402
from paper_2605_20977_b200.codec import (BandGroupCodec, GpuCodec, band_rows, gen_weights,  # noqa: E402
                                         make_cfg, split_banded, synth_latent)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="desk")
    ap.add_argument("--height", type=int, default=16)
    ap.add_argument("--width", type=int, default=16)
    ap.add_argument("--fidx", type=int, default=2)
    ap.add_argument("--lanes", type=int, default=32)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--same-device", action="store_true")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = 0 if a.same_device else int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    cfg = make_cfg(a.preset, a.height, a.width, lanes=a.lanes, hyper_lanes=16)
    blob = gen_weights(cfg, 1)
    frames = [synth_latent(cfg, 0, f) for f in range(a.fidx + 1)]
    payload = [None]
    if rank == 0:
        enc = BandGroupCodec(cfg, blob, [dev] * world)
        for f in frames[:a.fidx]:
            enc.push_frame(f)
        hyper, main, _ = enc.encode_frame(frames[a.fidx], fidx=a.fidx)
        enc.close()
        payload = [(hyper, main)]
    dist.broadcast_object_list(payload, src=0)
    hyper, main = payload[0]
    mine = split_banded(main, world)[rank]
    band = GpuCodec(cfg, blob, device=dev, band=rank, n_bands=world)
    pdist.link_band(band, dist)
    for f in frames[:a.fidx]:
        band.push_frame(f)
    dist.barrier()
    times = []
    for _ in range(a.steps):
        dist.barrier()
        t0 = time.perf_counter()
        y, bits = band.decode_frame(hyper, mine, fidx=a.fidx, advance=False)
        times.append(time.perf_counter() - t0)
    r0, r1 = band_rows(a.height, world, rank)
    parts = [None] * world if rank == 0 else None
    dist.gather_object((r0, r1, y[:, r0:r1].copy(), float(bits[1]), max(times)), parts, dst=0)
    if rank == 0:
        full = np.zeros_like(frames[a.fidx])
        for p0, p1, rows, _, _ in parts:
            full[:, p0:p1] = rows
        exact = bool(np.array_equal(full, frames[a.fidx]))
        res = {"bands": world, "grid": [a.height, a.width], "preset": a.preset,
               "same_device": a.same_device, "bit_exact": exact,
               "main_bits": sum(p[3] for p in parts),
               "host_ms_per_frame_max_over_ranks": 1e3 * max(p[4] for p in parts),
               "launches_per_band": band.last_launch_count()}
        print(json.dumps(res), flush=True)
        if a.out:
            json.dump(res, open(a.out, "w"))
        if not exact:
            sys.exit(1)
    band.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
