"""Copy-engine probe: how fast do the copy programs' copies run on this B200?

Times (CUDA events on a dedicated stream) several ways of moving the 56 MiB a
C2 rank ingests (56 fine chunks of 1 MiB, or 7 shards of 8 MiB):
  one_big        one 56 MiB cudaMemcpyAsync
  shards7        7 x 8 MiB in one ficco_copy_batch call (one copy per entry)
  chunks56       56 x 1 MiB in one batch
  rounds8x7      8 batches of 7 x 1 MiB (the fine-grain copy program shape)
  torch_copy     torch .copy_ of 8 x 7 MiB slices (reference point)
optionally while the tile kernel occupies every SM (``--busy``).
"""
import argparse
import ctypes as C
import json
import statistics
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
from paper_2512_10236_b200 import runtime  # noqa: E402


def batch(dsts, srcs, sizes, stream):
    n = len(dsts)
    lib = runtime.load_library()
    d = (C.c_void_p * n)(*dsts)
    s = (C.c_void_p * n)(*srcs)
    z = (C.c_size_t * n)(*sizes)
    runtime.check(lib.ficco_copy_batch(d, s, z, n, C.c_void_p(stream.cuda_stream)))


def timeit(fn, stream, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--busy", action="store_true")
    args = ap.parse_args()
    runtime.load_library()
    MiB = 1 << 20
    src = torch.empty(64 * MiB, dtype=torch.uint8, device="cuda")
    dst = torch.empty(64 * MiB, dtype=torch.uint8, device="cuda")
    src.fill_(3)
    s = torch.cuda.Stream()
    sp, dp = src.data_ptr(), dst.data_ptr()
    res = {}
    with torch.cuda.stream(s):
        res["one_big_56MiB"] = timeit(lambda: batch([dp], [sp], [56 * MiB], s), s)
        res["shards7x8MiB"] = timeit(lambda: batch([dp + i * 8 * MiB for i in range(7)],
                                                   [sp + i * 8 * MiB for i in range(7)], [8 * MiB] * 7, s), s)
        res["chunks56x1MiB"] = timeit(lambda: batch([dp + i * MiB for i in range(56)],
                                                    [sp + i * MiB for i in range(56)], [MiB] * 56, s), s)

        def rounds():
            for r in range(8):
                batch([dp + (r * 7 + i) * MiB for i in range(7)], [sp + (r * 7 + i) * MiB for i in range(7)],
                      [MiB] * 7, s)
        res["rounds8x7x1MiB"] = timeit(rounds, s)

        def single_copies():
            for i in range(56):
                batch([dp + i * MiB], [sp + i * MiB], [MiB], s)
        res["56_single_1MiB"] = timeit(single_copies, s)
        res["torch_copy_56MiB"] = timeit(lambda: dst[:56 * MiB].copy_(src[:56 * MiB]), s)
    for k, v in list(res.items()):
        res[k] = {"us": round(v, 2), "GBps": round(56 * MiB / (v * 1e-6) / 1e9, 1)}
    print(json.dumps(res, indent=1))


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def sweep():
    """Single-copy latency vs size, and k concurrent 1 MiB copies on k streams."""
    runtime.load_library()
    MiB = 1 << 20
    src = torch.empty(128 * MiB, dtype=torch.uint8, device="cuda").fill_(1)
    dst = torch.empty(128 * MiB, dtype=torch.uint8, device="cuda")
    s0 = torch.cuda.Stream()
    out = {"size_sweep": {}, "streams": {}}
    for kb in (64, 256, 512, 1024, 2048, 4096, 8192, 16384, 65536):
        n = kb * 1024
        us = timeit(lambda: batch([dst.data_ptr()], [src.data_ptr()], [n], s0), s0)
        out["size_sweep"][f"{kb}KiB"] = {"us": round(us, 2), "GBps": round(n / (us * 1e-6) / 1e9, 1)}
    streams = [torch.cuda.Stream() for _ in range(16)]
    main = torch.cuda.current_stream()
    for k in (1, 2, 4, 7, 8, 14, 16):
        for per in (1, 8):
            def run():
                ev = torch.cuda.Event()
                ev.record(main)
                for i in range(k):
                    streams[i].wait_event(ev)
                    for j in range(per):
                        off = (i * per + j) % 120 * MiB
                        batch([dst.data_ptr() + off], [src.data_ptr() + off], [MiB], streams[i])
                for i in range(k):
                    e2 = torch.cuda.Event()
                    e2.record(streams[i])
                    main.wait_event(e2)
            us = timeit(run, main)
            out["streams"][f"{k}x{per}x1MiB"] = {"us": round(us, 2), "GBps": round(k * per * MiB / (us * 1e-6) / 1e9, 1)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "sweep":
    sweep()


def hidden():
    """Separate host enqueue cost from GPU execution: enqueue behind a GPU sleep."""
    import time
    runtime.load_library()
    MiB = 1 << 20
    src = torch.empty(128 * MiB, dtype=torch.uint8, device="cuda").fill_(1)
    dst = torch.empty(128 * MiB, dtype=torch.uint8, device="cuda")
    main = torch.cuda.current_stream()
    streams = [torch.cuda.Stream() for _ in range(8)]
    out = {}
    for label, n, size, nstreams, per_call in [("56x1MiB_1stream_1batch", 56, MiB, 1, 56),
                                               ("56x1MiB_1stream_56calls", 56, MiB, 1, 1),
                                               ("56x1MiB_7streams", 56, MiB, 7, 1),
                                               ("56x1MiB_7streams_batch8", 56, MiB, 7, 8),
                                               ("7x8MiB_7streams", 7, 8 * MiB, 7, 1),
                                               ("7x8MiB_1stream", 7, 8 * MiB, 1, 7),
                                               ("1x56MiB", 1, 56 * MiB, 1, 1),
                                               ("memcpyAsync_56x1MiB_7streams", 56, MiB, 7, -1)]:
        res = []
        for rep in range(6):
            torch.cuda.synchronize()
            torch.cuda._sleep(20_000_000)  # ~10 ms of GPU time to hide the host enqueue
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(main)
            t0 = time.perf_counter()
            per_stream = n // nstreams
            for si in range(nstreams):
                s = streams[si]
                s.wait_event(a)
                i0 = si * per_stream
                if per_call == -1:
                    for i in range(i0, i0 + per_stream):
                        with torch.cuda.stream(s):
                            dst[i * size:(i + 1) * size].copy_(src[i * size:(i + 1) * size], non_blocking=True)
                else:
                    for j in range(i0, i0 + per_stream, per_call):
                        m = min(per_call, i0 + per_stream - j)
                        batch([dst.data_ptr() + (j + q) * size for q in range(m)],
                              [src.data_ptr() + (j + q) * size for q in range(m)], [size] * m, s)
            host_us = (time.perf_counter() - t0) * 1e6
            for si in range(nstreams):
                e = torch.cuda.Event()
                e.record(streams[si])
                main.wait_event(e)
            b.record(main)
            b.synchronize()
            res.append((a.elapsed_time(b) * 1e3, host_us))
        res = res[2:]
        gpu = statistics.median(r[0] for r in res)
        out[label] = {"gpu_us": round(gpu, 2), "host_us": round(statistics.median(r[1] for r in res), 1),
                      "GBps": round(n * size / (gpu * 1e-6) / 1e9, 1)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "hidden":
    hidden()
