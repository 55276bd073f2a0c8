"""Fresh-context extractions at C3 (the bench's e2e pattern): host time, device phases and kernel launches per
call, to separate allocation / retry costs from the device work."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2412_13576_b200 import maple
    from synth import c3
    inst = c3()
    maple.load()
    stream = torch.cuda.Stream()
    for it in range(5):
        t0 = time.perf_counter()
        ctx = maple.Context(inst.A, inst.l, inst.u)
        ctx.set_stream(stream.cuda_stream)
        t1 = time.perf_counter()
        ds = ctx.extract(inst.n_starts, inst.steps, inst.lr, inst.seed)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        free, total = torch.cuda.mem_get_info()
        print(f"iter {it}: create {1e3*(t1-t0):.1f} ms extract {1e3*(t2-t1):.1f} ms launches {ctx.launches()} "
              f"rows {ds.size} free {free/1e9:.1f} GB timings {ctx.timings()}", flush=True)
        ds.free()
        ctx.close()


if __name__ == "__main__":
    main()
