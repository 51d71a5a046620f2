"""Run tests/test_gpu_sharded_two_ranks.py's rank body in two processes with faulthandler
stack dumps on a hang (diagnostics)."""
import faulthandler
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def child(rank, port, kind, q):
    faulthandler.dump_traceback_later(45, exit=True)
    import time

    import torch

    import paper_2208_05321_b200.distributed as D
    import test_gpu_sharded_two_ranks as t
    orig = D.Router.route

    def route(self, ids):
        t0 = time.time()
        print(f"[{rank}] route n={ids.numel()} stream={torch.cuda.current_stream()}", file=sys.stderr, flush=True)
        r = orig(self, ids)
        print(f"[{rank}] route done {time.time() - t0:.3f}s u={r[0].numel()} sc={r[2]}", file=sys.stderr, flush=True)
        return r

    D.Router.route = route

    def wrap(cls, name):
        f = getattr(cls, name)

        def g(*a, **k):
            t0 = time.time()
            print(f"[{rank}] {name} ...", file=sys.stderr, flush=True)
            r = f(*a, **k)
            torch.cuda.synchronize()
            print(f"[{rank}] {name} done {time.time() - t0:.3f}s", file=sys.stderr, flush=True)
            return r
        setattr(cls, name, g)

    for nm in ("prepare", "pool", "backward"):
        wrap(D.CudaShard, nm)
    for nm in ("pool", "grads"):
        wrap(D.Router, nm)
    if os.environ.get("SIDE_STREAM"):
        with torch.cuda.stream(torch.cuda.Stream(0)):
            t._rank_main(rank, 2, port, kind, False, q)
    else:
        t._rank_main(rank, 2, port, kind, False, q)


if __name__ == "__main__":
    import torch.multiprocessing as mp

    import test_gpu_sharded_two_ranks as t
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = t._free_port()
    ps = [ctx.Process(target=child, args=(r, port, sys.argv[1] if len(sys.argv) > 1 else "row", q)) for r in range(2)]
    for p in ps:
        p.start()
    for _ in range(2):
        try:
            r = q.get(timeout=90)
            print("got", r[0], type(r[1]), (r[1] if isinstance(r[1], str) else ""))
        except Exception as e:
            print("timeout", e)
    for p in ps:
        p.join(timeout=30)
        print("exit", p.exitcode)
