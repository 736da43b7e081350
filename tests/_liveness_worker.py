"""Worker for tests/test_gpu_liveness.py: Stream-K launches on several streams at once.

Each of S streams owns a plan (hence its own per-stream workspace); every round launches
all of them back to back, so Stream-K grids whose reducers spin on peer flags run
concurrently with other Stream-K grids (and, under the test, another process).  Exits 0
when every result is bitwise equal to the float64 product of the integer inputs.
"""

import sys

import torch


def main(rounds: int, streams: int, seed: int) -> int:
    sys.path.insert(0, sys.argv[4] if len(sys.argv) > 4 else ".")
    import paper_2408_11417_b200 as sk

    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    m, n, k = 512, 512, 8192
    a = torch.randint(-8, 9, (m, k), generator=gen, device="cuda", dtype=torch.int8)
    b = torch.randint(-8, 9, (k, n), generator=gen, device="cuda", dtype=torch.int8)
    want = a.double() @ b.double()
    ab, bb = a.to(torch.bfloat16), b.to(torch.bfloat16)
    lo, hi = torch.cuda.Stream.priority_range()
    sts = [torch.cuda.Stream(priority=lo if i % 2 else hi) for i in range(streams)]
    plans = [sk.GemmPlan(ab, bb, torch.zeros(m, n, device="cuda"),
                         sk.Policy.all_stream_k() if i % 2 else sk.Policy.hybrid(1),
                         sk.TileShape(128, 128, 64) if i % 2 else sk.TileShape(256, 256, 64))
             for i in range(streams)]
    for st in sts:
        st.wait_stream(torch.cuda.current_stream())
    for _ in range(rounds):
        for p, st in zip(plans, sts):
            p.launch(stream=st)
    torch.cuda.synchronize()
    for p in plans:
        if not torch.equal(p.c.double(), want):
            print("mismatch", flush=True)
            return 1
    print("ok", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])))
