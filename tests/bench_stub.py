"""A CPU stand-in for bench.py's native engine (bench.NativeEngine), used only by
tests/test_bench_launcher.py to run bench.py's real multi-rank control flow (launcher, gloo
process group, warm-up, barriers, timed steps, MAX-reduced time, SUM-reduced counters, rank-0 line)
on a machine without GPUs.  It decodes nothing: each frame's counters are a fixed function of its
global frame id, so the expected totals do not depend on how the frames are sharded."""
import time

import torch

import bench
import synth

SLEEP_S = 0.03   # per step and rank index + 1: the slowest rank sets the reported time


def frame_counters(fid):
    """[frames, successes, frames with bit errors, undetected, iterations] of global frame fid."""
    succ = int(fid % 3 != 0)
    err = int(fid % 3 == 0 or fid % 7 == 0)
    return [1, succ, err, int(succ and err), fid % 11]


class StubEngine:
    backend = "gloo"
    device_id = None

    def __init__(self, args, world, rank, local):
        self.args, self.world, self.rank = args, world, rank

    def prepare(self):
        self.names = bench.WORKLOADS[self.args.workload]
        self.shards = [bench.shard(synth.workload(n).frames, self.rank, self.world) for n in self.names]
        self.launches_per_step = 0
        return list(self.names)

    def zeros(self, shape):
        return torch.zeros(shape, dtype=torch.int64)

    def step(self, counters, record):
        counters.zero_()
        for i, (a, b) in enumerate(self.shards):
            counters[i] = torch.tensor([sum(v) for v in zip(*[frame_counters(f) for f in range(a, b)])],
                                       dtype=torch.int64)
        time.sleep(SLEEP_S * (self.rank + 1))

    def sync(self):
        pass

    def clear_records(self):
        pass

    def start_timer(self):
        self.t0 = time.perf_counter()

    def stop_timer(self):
        return (time.perf_counter() - self.t0) * 1000.0

    def decode_ms(self, i):
        return 0.0

    def payload_bits(self, i):
        return 100

    def extras(self, c, ms_total, per_wl):
        return {"dtype": "none (stub)", "rank_slept_ms_per_step": 1000 * SLEEP_S * self.world}
