"""Experiment: does issuing row groups of the step on separate CUDA streams
(so one group's kernel fills another's tail) shorten the 1.4B step?
usage: python tools/exp_streams.py [groups ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import workload  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    cfg = workload.CONFIGS["1.4b"]
    D = bench.setup_native(torch, cfg, 0, 1, dev)
    base = bench.Step(torch, cfg, D, dev, 1, None)

    def time_it(fn, n=30, w=5):
        for _ in range(w):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    print("1 stream      : %.3f ms" % time_it(base.kernels), flush=True)
    for G in [int(g) for g in sys.argv[1:]] or [2, 4]:
        rg = cfg.R // G
        subs = []
        for g in range(G):
            sl = slice(g * rg, (g + 1) * rg)
            Dg = dict(D, T={k: v[sl] for k, v in D["T"].items()}, pos=D["pos"][sl])
            cg = workload.Shape(cfg.name, rg, cfg.L, cfg.Dn, cfg.N, cfg.K, cfg.dtype)
            subs.append(bench.Step(torch, cg, Dg, dev, 1, None))
        streams = [torch.cuda.Stream() for _ in range(G)]

        def run():
            main_s = torch.cuda.current_stream()
            e0 = torch.cuda.Event()
            e0.record(main_s)
            ends = []
            for s, st in zip(streams, subs):
                s.wait_event(e0)
                with torch.cuda.stream(s):
                    st.kernels()
                    e = torch.cuda.Event()
                    e.record(s)
                    ends.append(e)
            for e in ends:
                main_s.wait_event(e)
            tot = subs[0].pg.flat
            for st in subs[1:]:
                tot.add_(st.pg.flat)

        print("%d streams x %d rows: %.3f ms" % (G, rg, time_it(run)), flush=True)


if __name__ == "__main__":
    main()
