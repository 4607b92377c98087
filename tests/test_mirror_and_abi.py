"""CPU-side checks of the product library (no GPU calls):

* libpbkv.so loads and exports every symbol include/pbkv.h declares;
* without a B200 the context cannot be created (no CPU fallback);
* the host RadixMirror reproduces the reference CacheTree field by field
  for the same operation stream (random streams and the synthetic generator).
"""
import ctypes as C

import numpy as np
import pytest

import workloads as WL
from oracle import RefTree, have_ref
from paper_2605_06472_b200 import _abi
from paper_2605_06472_b200.api import HostTree, PbkvError, Policy, ValidationError


def test_library_exports_every_declared_symbol():
    L = C.CDLL(_abi.LIB_PATH)
    syms = _abi.exported_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert _abi.lib().pbkv_abi_version() == 2


def test_no_cpu_fallback_without_gpu():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is visible")
    except Exception:
        pass
    with pytest.raises(PbkvError) as ei:
        Policy(num_agents=4)
    assert ei.value.status == _abi.PBKV_ECUDA


def test_ctx_validates_score_params_first():
    with pytest.raises(ValidationError, match="gamma must be in"):
        Policy(num_agents=4, k=3, gamma=1.0)
    with pytest.raises(ValidationError, match="lookahead horizon"):
        Policy(num_agents=4, k=0)


FIELDS = ["parent", "len", "tier", "retired", "last_access", "ever_tagged", "score", "device_children", "depth"]


def assert_same_tree(a, b):
    assert a.n_nodes == b.n_nodes and a.n_entries == b.n_entries
    for f in FIELDS:
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(a.acc_off, b.acc_off)
    assert np.array_equal(a.acc_wf[: a.n_entries], b.acc_wf[: b.n_entries])
    assert np.array_equal(a.acc_bits[: a.n_entries], b.acc_bits[: b.n_entries])
    assert a.scalars == b.scalars


@pytest.mark.skipif(not have_ref(), reason="reference oracle not built")
@pytest.mark.parametrize("seed", range(60))
def test_mirror_matches_reference_cachetree(seed):
    rng = np.random.default_rng(7000 + seed)
    ops, live = WL.random_tree_ops(rng, n_ops=int(rng.integers(5, 80)), n_wf=int(rng.integers(2, 10)),
                                   agents=int(rng.integers(1, 6)), alphabet=3, max_len=8)
    ref = RefTree(1 << 20, int(rng.integers(0, 40)) if seed % 3 == 0 else 1 << 20)
    ref.apply_ops(ops.words)
    for d in WL.legal_demotions(ref.export(), rng, 0.25):
        ops.demote(d)
    # promotions of some host nodes whose parent is device
    ref = RefTree(1 << 20, 1 << 20)
    ref.apply_ops(ops.words)
    soa = ref.export()
    for i in range(1, soa.n_nodes):
        if soa.tier[i] == 1 and soa.tier[soa.parent[i]] == 0 and rng.random() < 0.3:
            ops.promote(i)
    for i in range(1, soa.n_nodes):
        if rng.random() < 0.1:
            ops.set_score(i, float(rng.random()))
    ref = RefTree(1 << 20, 1 << 20)
    ref.apply_ops(ops.words)
    mine = HostTree(1 << 20, 1 << 20)
    mine.apply_ops(ops.words)
    assert_same_tree(mine.export(), ref.export())
    for w in live:
        assert mine.touched(w) == ref.touched(w)


@pytest.mark.skipif(not have_ref(), reason="reference oracle not built")
@pytest.mark.parametrize("n_nodes,n_wf", [(3000, 64), (10000, 256)])
def test_synthetic_generator_matches_reference(n_nodes, n_wf):
    ref = RefTree()
    ref.synth(n_nodes=n_nodes, n_workflows=n_wf)
    mine = HostTree()
    mine.synth(n_nodes=n_nodes, n_workflows=n_wf)
    a, b = mine.export(), ref.export()
    assert_same_tree(a, b)
    # the generator's shape: ~30% retired, E/N well below 1
    assert 0.2 < b.retired[1:].mean() < 0.4
    assert 0.4 < b.n_entries / b.n_nodes < 1.0


def test_mirror_errors_are_validation_errors():
    t = HostTree(100, 100)
    with pytest.raises(ValidationError, match="demote needs a device node"):
        t.apply_ops([4, 0])
    with pytest.raises(ValidationError, match="insert_suffix without room"):
        from paper_2605_06472_b200.ops import OpStream

        t.apply_ops(OpStream().insert(list(range(200)), 1, 0).words)


def test_round_victims_behaves_like_list_of_lists():
    import numpy as np

    from paper_2605_06472_b200.api import RoundVictims

    rv = RoundVictims(np.array([5, 6, 7, 9], dtype=np.int32), np.array([0, 2, 2, 4], dtype=np.int64))
    want = [[], [5, 6], [], [7, 9]]
    assert rv == want and list(rv) == want and len(rv) == 4 and rv[-1] == [7, 9]
    assert rv != [[], [5, 6], [], [7]] and rv != [[5], [6], [], [7, 9]] and rv != want[:3]
    assert RoundVictims(np.zeros(0, np.int32), np.zeros(0, np.int64)) == []
