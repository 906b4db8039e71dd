"""A/B of the host-edge-list bridges call (ettg_bridges, int64 edges -> host
mask) on config D: ETTG_NARROW (u32 narrowing on host threads), ETTG_BR_STREAM
(hooking overlapped with the upload), ETTG_MASK_BITS (bit-packed mask D2H);
pinned and pageable buffers (dev aid)."""
import itertools, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
L = _lib.lib()
g, truth = ett.road_like_graph(5657, 5657, 6, 3, 20_761, 5)
m = g.m()
pin_e = torch.from_numpy(np.ascontiguousarray(g.edges, dtype=np.int64)).pin_memory()
pin_m = torch.empty(m, dtype=torch.uint8).pin_memory()
pg_m = np.empty(m, np.uint8)
combos = list(itertools.product(["0", "1"], ["0", "1"], ["0", "1"]))
for rnd in range(2):
    for (nar, stream, bits) in combos:
        os.environ.update(ETTG_NARROW=nar, ETTG_BR_STREAM=stream, ETTG_MASK_BITS=bits)
        for kind, e, mk in (("pinned", pin_e.numpy(), pin_m.numpy()), ("pageable", g.edges, pg_m)):
            ts = []
            for _ in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                _lib.check(L.ettg_bridges(e.ctypes.data, g.n, m, 0, mk.ctypes.data, None))
                ts.append(time.perf_counter() - t0)
            ok = np.array_equal(mk, truth)
            print(rnd, f"narrow={nar} stream={stream} bits={bits} {kind:8s} min {min(ts)*1e3:.2f} "
                  f"med {np.median(ts)*1e3:.2f} ms ok={ok}", flush=True)
