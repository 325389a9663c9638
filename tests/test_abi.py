"""CPU suite: the C-ABI library builds, loads and exports every symbol the
header declares; ctypes layouts match the C compiler's; host-side pieces
(corpus generator, packer) are exact; the device entry points fail loudly
without a GPU instead of falling back to the CPU."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

from oracle import bindings
from paper_2602_20826_b200 import _abi, _lib
from paper_2602_20826_b200.batch import combine_status, pack
from tests import helpers

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dagsched_b200.h")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        subprocess.run(["make", "-C", ROOT, "product"], check=True, capture_output=True)
    return _lib.lib()


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(ds_\w+)\(", text, re.M)))


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 12
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (ds_\w+)", out))
    assert set(names) <= exported, set(names) - exported
    for n in names:
        assert hasattr(lib, n)


def test_struct_layouts_match_c():
    structs = ["ds_platform", "ds_dag_batch", "ds_dag_batch16", "ds_results", "ds_gen_config", "ds_entity_rec",
               "ds_group_rec", "ds_scheme_out"]
    src = '#include <stdio.h>\n#include "dagsched_b200.h"\nint main(){\n' + "".join(
        f'printf("{s} %zu\\n", sizeof({s}));\n' for s in structs) + "return 0;}\n"
    with tempfile.TemporaryDirectory() as d:
        with open(os.path.join(d, "s.c"), "w") as f:
            f.write(src)
        exe = os.path.join(d, "s")
        subprocess.run(["gcc", "-I", os.path.dirname(HEADER), os.path.join(d, "s.c"), "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True).stdout
    sizes = dict(line.split() for line in out.strip().splitlines())
    for s in structs:
        assert int(sizes[s]) == C.sizeof(getattr(_abi, s)), s


@pytest.mark.parametrize("cfg", [dict(seed=1), dict(seed=12345, avg_load=200, max_width=16),
                                 dict(seed=3, integer_loads=False, avg_load=5),
                                 dict(seed=11, exact_mean=True, integer_loads=False, avg_load=7),
                                 dict(seed=4, t_min="1/2", avg_load=9)])
def test_host_generator_matches_reference_generator(lib, cfg):
    """ds_corpus_generate (product, host C++) is bit-identical to the
    reference's generate_corpus (generator.cpp:24-108)."""
    chk = bindings.Checker("ref" if bindings.available("ref") else "oracle")
    want = chk.generate(3000, **cfg).pack()
    got = _lib.Corpus(3000, **cfg).batch()
    for k in ("node_off", "edge_off", "load_num", "load_den", "edges"):
        assert np.array_equal(getattr(got, k), getattr(want, k)), k


def test_generator_rejects_bad_config(lib):
    with pytest.raises(_lib.DagschedError):
        _lib.Corpus(10, depth_min=1)
    with pytest.raises(_lib.DagschedError):
        _lib.Corpus(10, load_jitter=2.0)
    with pytest.raises(_lib.DagschedError):
        _lib.Corpus(0)


def test_packer_status_order():
    # dag.cpp order: empty, duplicate id, load, edges (first in sorted order), cycle/sources/sinks
    b = pack([([], []), ([(1, 1), (1, 2)], []), ([(0, 1)], [(0, 9)]), ([(0, 1), (1, 1)], [(1, 1), (0, 5)]),
              ([(0, "1/2")], [(0, 7)])])
    assert list(b.pack_status) == [_abi.DS_E_EMPTY, _abi.DS_E_DUP_ID, _abi.DS_E_EDGE, _abi.DS_E_EDGE,
                                   _abi.DS_E_EDGE]
    dev = np.array([0, 0, 0, 0, _abi.DS_E_LOAD], np.int32)
    assert list(combine_status(b.pack_status, dev))[-1] == _abi.DS_E_LOAD  # load check precedes edges


def test_fixture_packing_matches_raw():
    for case in helpers.fixtures():
        if case["status"] == 0:
            a, b = helpers.fixture_batch(case), helpers.fixture_raw_batch(case)
            assert np.array_equal(a.load_num, b.load_num)
            assert sorted(set(b.edges.tolist())) == a.edges.tolist()


def test_device_path_fails_loudly_without_gpu(lib):
    if _lib.device_count() > 0:
        pytest.skip("GPU present")
    b = pack([([1, 2, 1], [(0, 1), (1, 2)])])
    with pytest.raises(_lib.DagschedError):
        _lib.analyze(b, 8)


def test_compact16_packing_roundtrip():
    """DagBatch.compact16: 16-bit loads and from << 8 | to edges, host side."""
    from paper_2602_20826_b200.batch import pack
    from paper_2602_20826_b200 import workloads
    b = pack([workloads.make_example_task(), workloads.c1_fork_join()])
    assert b.compact16_ok()
    load16, edges16 = b.compact16()
    assert load16.dtype == np.uint16 and edges16.dtype == np.uint16
    assert np.array_equal(load16.astype(np.int64), b.load_num)
    assert np.array_equal(((edges16 >> 8).astype(np.uint32) << 16) | (edges16 & 0xFF), b.edges)
    big = pack([([(0, 70000), (1, 1)], [(0, 1)])])
    assert not big.compact16_ok()


def test_compact16_entry_validates_arguments(lib):
    """ds_analyze_batch16 rejects NULL arrays with DS_EINVAL before touching a
    device, and without a GPU the compute call fails loudly (no CPU path)."""
    L = _lib.lib()
    b = pack([([1, 2, 1], [(0, 1), (1, 2)])])
    st = np.zeros(1, np.int32)
    bo = np.zeros((1, 10), np.int64)
    r = _abi.ds_results(st.ctypes.data, bo.ctypes.data, None)
    pl = _lib.platform(8)
    bad = _abi.ds_dag_batch16(1, b.node_off.ctypes.data, b.edge_off.ctypes.data, None, None)
    assert L.ds_analyze_batch16(C.byref(bad), C.byref(pl), _abi.DS_M_ALL, C.byref(r), 0) == _abi.DS_EINVAL
    if _lib.device_count() == 0:
        with pytest.raises(_lib.DagschedError):
            _lib.analyze16(b, 8)


def test_scheme_self_checks_reject_cycles_and_oversubscription():
    """scheduler.cpp:389-424: an augmented-graph cycle or a group holding more
    than M SMs is a scheduler bug -> DS_EINVARIANT (logic_error there)."""
    from fractions import Fraction as F

    from paper_2602_20826_b200 import scheme as S

    def ent(o, m=1):
        return S.Entity(S.EntityId(o), F(1), m, F(1), 0, False)

    a, b = ent(0), ent(1)
    g = S.Group(0, [a, b], [], 0, F(1), a.id, 0)
    ok = S.Scheme(2, F(1), [g], [], [], [a, b], [0, 0], [0, 0], 1, {})
    b.preds = [a.id]
    S.verify(ok)  # a -> b, 2 SMs on M = 2
    a.preds = [b.id]
    with pytest.raises(_lib.DagschedError) as e:
        S.verify(ok)
    assert e.value.code == _abi.DS_EINVARIANT and "cycle" in str(e.value)
    a.preds = []
    over = S.Scheme(1, F(1), [g], [], [], [a, b], [0, 0], [0, 0], 1, {})
    with pytest.raises(_lib.DagschedError) as e:
        S.verify(over)
    assert "exceeds the device" in str(e.value)


def test_triangular_packer_roundtrip():
    """batch.tri(): node v's predecessor bits v(v-1)/2 + u decode back to the
    DAG's (deduplicated, sorted) edge list (host only)."""
    from paper_2602_20826_b200 import _lib
    b = _lib.Corpus(3000, seed=4).batch()
    load, adj_off, adj = b.tri()
    assert np.array_equal(load, b.load_num.astype(np.uint16))
    for d in range(0, 3000, 97):
        n0, n1 = int(b.node_off[d]), int(b.node_off[d + 1])
        e0, e1 = int(b.edge_off[d]), int(b.edge_off[d + 1])
        w = adj[adj_off[d]:adj_off[d + 1]]
        n = n1 - n0
        got = [(u << 16) | v for u in range(n) for v in range(u + 1, n)
               if (int(w[(v * (v - 1) // 2 + u) >> 5]) >> ((v * (v - 1) // 2 + u) & 31)) & 1]
        assert got == sorted(set(int(x) for x in b.edges[e0:e1]))
