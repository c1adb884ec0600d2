"""Debug: two ranks (one process each, both on cuda:0) run a k=2 LU plan; report which tiles
differ from the oracle, in final-writer task order.  python tools/debug_multirank_lu.py N NB [launches] [push]"""
import math
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, q, n, b, launches, push, single):
    import torch.distributed as dist

    import paper_1402_6601_b200 as H
    from paper_1402_6601_b200 import runtime
    from oracle import tiles as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ib = 128
        g = H.gen_family("lu", n // b, b, ib)
        plat = H.build_platform(world, world, world, link_bandwidth=7.7e11, link_latency=3e-6,
                                switch_cap=math.inf, p2p=True)
        plan = H.make_plan(g, plat, H.make_scheduler("dada", alpha=0.5, cp=True),
                           H.PerfModel(H.default_timing_table(b, ib)))
        A = O.general_matrix(n, 3)
        img = runtime.to_tile_major(A, g)
        out = np.full_like(img, np.nan)
        ex = runtime.DistributedExecutor(g, plat, plan, img, out, rank=rank, world=world, device=0, push=push)
        for _ in range(launches):
            ex.launch(0)
            if single:
                ex.wait()
        ex.wait()
        st = ex.info()
        ex.close()
        q.put((rank, out, st.bytes_h2d, st.bytes_d2d))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def main():
    import torch.multiprocessing as mp

    import paper_1402_6601_b200 as H
    from paper_1402_6601_b200 import runtime
    from oracle import tiles as O

    n, b = int(sys.argv[1]), int(sys.argv[2])
    launches = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    push = (sys.argv[4] == "1") if len(sys.argv) > 4 else True
    single = (sys.argv[5] == "1") if len(sys.argv) > 5 else True
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q, n, b, launches, push, single)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(2)], key=lambda r: r[0])
    for p in procs:
        p.join(60)
    ib = 128
    g = H.gen_family("lu", n // b, b, ib)
    plat = H.build_platform(2, 2, 2, link_bandwidth=7.7e11, link_latency=3e-6, switch_cap=math.inf, p2p=True)
    plan = H.make_plan(g, plat, H.make_scheduler("dada", alpha=0.5, cp=True), H.PerfModel(H.default_timing_table(b, ib)))
    merged = np.where(np.isnan(res[0][1]), res[1][1], res[0][1])
    A = O.general_matrix(n, 3)
    T = {d: np.asfortranarray(t) for d, t in O.tiles_of(A, g.layout).items()}
    O.run_tasks(g, T, side={})
    offs = np.cumsum([0] + [s // 8 for s in g.sizes])
    final_writer = {}
    for t in range(len(g)):
        for d, m in g.tasks[t].accesses:
            if d in g.layout.tiles and "W" in m.value:
                final_writer[d] = t
    rows = []
    for d, (i, j) in g.layout.tiles.items():
        got = merged[offs[d]:offs[d + 1]].reshape(b, b, order="F")
        rel = float(np.abs(got - T[d]).max() / np.abs(T[d]).max())
        w = final_writer.get(d, -1)
        rows.append((w, (i, j), rel, g.tasks[w].kind if w >= 0 else "-", int(plan.worker[w]) if w >= 0 else None))
    rows.sort()
    bad = [r for r in rows if r[2] > 1e-11]
    print(f"n={n} nb={b} launches={launches} push={push} single={single}: {len(bad)} bad tiles of {len(rows)}; "
          f"bytes h2d {sum(r[2] for r in res)} vs {plan.bytes_h2d}, d2d {sum(r[3] for r in res)} vs {plan.bytes_d2d}")
    for r in bad[:12]:
        print("  ", r)


if __name__ == "__main__":
    main()
