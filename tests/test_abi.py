"""CPU: the C-ABI library loads, exports every declared symbol, and its
host-side entry points (cluster_bfs, load_partition core) are bit-exact."""
import ctypes
import re

import numpy as np
import pytest

from conftest import ROOT

from paper_2305_17408_b200 import _lib


def header_symbols():
    text = (ROOT / "include" / "adaptgear_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|uint64_t|const char \*)\s*(ag_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    assert lib.ag_abi_version() == 1


def test_no_device_is_reported_without_gpu():
    lib = _lib.load()
    assert lib.ag_device_sm_count() >= 0


def test_product_refuses_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="CUDA device"):
        _lib.device()


def _bfs(V, dst, src, B):
    dst = np.ascontiguousarray(dst, np.int32)
    src = np.ascontiguousarray(src, np.int32)
    comm = np.empty(V, np.int64)
    perm = np.empty(V, np.int64)
    _lib.call("ag_cluster_bfs", V, dst.size, _lib.host_ptr(dst), _lib.host_ptr(src), B,
              _lib.host_ptr(comm), _lib.host_ptr(perm))
    return comm, perm


def test_cluster_bfs_host_bit_exact(reorder_golden):
    z = reorder_golden
    n = 0
    for i in z.cases("r"):
        p = f"r{i}_"
        comm, perm = _bfs(int(z[p + "V"]), z[p + "dst"], z[p + "src"], int(z[p + "B"]))
        assert np.array_equal(comm, z[p + "community"]), i
        assert np.array_equal(perm, z[p + "perm"]), i
        n += 1
    assert n >= 30


def test_cluster_bfs_host_vs_oracle_random(rng):
    from oracle import ref_numpy as R
    from conftest import random_graph_arrays
    for _ in range(40):
        V, d, s, _ = random_graph_arrays(rng, num_vertices=int(rng.integers(2, 200)))
        if rng.integers(2):
            d, s, _ = R.gcn_normalize(V, d, s)
        else:
            d, s, _ = R.canonical(V, d, s)
        B = int(rng.integers(1, 33))
        comm, perm = _bfs(V, d, s, B)
        c2, p2 = R.cluster_bfs(V, d, s, B)
        assert np.array_equal(comm, c2) and np.array_equal(perm, p2)


def test_cluster_bfs_rejects_bad_comm_size():
    with pytest.raises(ValueError):
        _bfs(2, [1], [0], 0)


def test_partition_from_ids_bit_exact(reorder_golden):
    z = reorder_golden
    for i in range(4):
        ids = np.ascontiguousarray(z[f"lp{i}_ids"], np.int64)
        comm = np.empty(ids.size, np.int64)
        perm = np.empty(ids.size, np.int64)
        _lib.call("ag_partition_from_ids", ids.size, _lib.host_ptr(ids), int(z[f"lp{i}_B"]),
                  _lib.host_ptr(comm), _lib.host_ptr(perm))
        assert np.array_equal(comm, z[f"lp{i}_community"])
        assert np.array_equal(perm, z[f"lp{i}_perm"])


def test_load_partition_errors(tmp_path):
    from paper_2305_17408_b200 import load_partition
    f = tmp_path / "p.txt"
    f.write_text("0\n-1\n")
    with pytest.raises(ValueError):
        load_partition(f, 2)
    f.write_text("0\nx\n")
    with pytest.raises(ValueError, match=":2:"):
        load_partition(f, 2)
    f.write_text("0\n" * 5)
    p = load_partition(f, 2)
    assert p.community_of.max() == 2


def test_edge_list_errors(tmp_path):
    from paper_2305_17408_b200 import EdgeListError, load_edge_list
    f = tmp_path / "g.txt"
    f.write_text("0 1\njunk\n")
    with pytest.raises(EdgeListError, match=":2:"):
        load_edge_list(f)
    f.write_text("# nothing\n")
    with pytest.raises(EdgeListError, match="no edges"):
        load_edge_list(f)
    f.write_text("0 -3\n")
    with pytest.raises(EdgeListError):
        load_edge_list(f)


def test_cluster_bfs_host_bit_exact_at_config_scale():
    """cluster_bfs at BASELINE scale (C2 pubmed-shaped, C3 ogbn-arxiv-shaped
    graphs from the numpy generator twin): the host C++ partition's digests
    equal the unmodified reference's (tests/golden/make_bfs_golden.py)."""
    import hashlib
    import json
    import pathlib
    from oracle import synth
    gold = json.loads((pathlib.Path(__file__).parent / "golden" / "bfs_scale.json").read_text())

    def digest(a):
        return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()

    for case in gold["cases"]:
        (dst, src), _ = synth.community_graph(case["V"], case["E"], seed=0, **case["generator"])
        assert dst.size == case["edges_canonical"], case["name"]
        comm, perm = _bfs(case["V"], dst, src, case["comm_size"])
        assert digest(comm) == case["community_sha256"], case["name"]
        assert digest(perm) == case["perm_sha256"], case["name"]
