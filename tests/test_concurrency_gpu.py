"""Host threads share the library: the scratch arena (Lease) and the pinned
staging buffers serialise per device, handles are independent.  Several
threads run LCA queries, bridges, parsing and primitives at once on
pageable and pinned buffers; every result must equal its single-threaded
answer."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_mixed_calls_from_threads(ett):
    import torch
    t = ett.permute_labels(ett.grasp_tree(300_000, 4, 3), 5)
    idx = ett.inlabel_build(t)
    q = ett.sample_queries(t.n, 400_000, 7)
    want_lca = ett.answer_batch(idx, q, len(q))
    g, truth = ett.planted_bridge_graph(200_000, 1_200_000, 400, 4)
    text = ett.write_edge_list(g)
    want_parse = ett.parse_edge_list(text).edges
    succ = np.arange(1, 500_001, dtype=np.int64)
    succ[-1] = -1
    vals = np.arange(500_000, dtype=np.int64) % 7
    want_scan = np.concatenate([[0], np.cumsum(vals)[:-1]])
    pinned_q = torch.from_numpy(q.copy()).pin_memory()
    pinned_a = torch.empty(len(q), dtype=torch.int64).pin_memory()
    errors = []

    def work(k):
        try:
            for _ in range(3):
                kind = k % 5
                if kind == 0:
                    assert np.array_equal(ett.answer_batch(idx, q, 1000), want_lca)
                elif kind == 1:
                    assert np.array_equal(ett.tv_bridges(g).is_bridge, truth)
                elif kind == 2:
                    assert np.array_equal(ett.parse_edge_list(text).edges, want_parse)
                elif kind == 3:
                    assert np.array_equal(ett.list_scan(succ, vals, 0), want_scan)
                else:
                    ett.lib().ettg_lca_query(idx.handle, pinned_q.data_ptr(), len(q), len(q),
                                             pinned_a.data_ptr())
                    assert np.array_equal(pinned_a.numpy(), want_lca)
        except Exception as e:  # pragma: no cover - reported below
            errors.append((k, repr(e)))

    threads = [threading.Thread(target=work, args=(k,)) for k in range(10)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors


def test_device_pointer_to_host_entry_point_is_rejected(ett):
    import torch
    t = ett.permute_labels(ett.grasp_tree(100_000, 4, 3), 5)
    idx = ett.inlabel_build(t)
    d = torch.zeros(2 * 100_000, dtype=torch.int64, device="cuda")
    a = np.empty(100_000, np.int64)
    rc = ett.lib().ettg_lca_query(idx.handle, d.data_ptr(), 100_000, 100_000, a.ctypes.data)
    assert rc == 1 and b"device pointer" in ett.lib().ettg_last_error()
