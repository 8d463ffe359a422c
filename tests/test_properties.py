"""Property tests (hypothesis), the reference's own properties for the host side of the path:
index <-> config bijection (test_kernels.py:103-108), super-graph augmentation preserving the
feature multiset (test_graphs.py:154-163), and the host layout / encoder agreeing with the
oracle restatement on arbitrary specs and configs."""

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import kt_oracle as ko
from paper_2102_04199_b200 import graphs as pg
from paper_2102_04199_b200 import kernels as pk

OPS = pk.OP_TYPES
TEMPLATE = pg.build_super_template(OPS)


@st.composite
def specs(draw):
    op = draw(st.sampled_from(OPS))
    one_d = op in ("conv1d", "transpose1d")
    size = draw(st.integers(150, 600) if one_d else st.integers(7, 224))
    cin = draw(st.integers(32, 128) if one_d else st.integers(3, 128))
    cout = draw(st.integers(32, 512) if one_d else st.integers(16, 128))
    ks = draw(st.sampled_from((1, 3, 5, 7)))
    return pk.KernelSpec(op, size, cin, cout, ks, 3, 1)


@settings(max_examples=60, deadline=None)
@given(specs(), st.data())
def test_index_config_bijection(spec, data):
    space = pk.build_knob_space(spec)
    i = data.draw(st.integers(0, space.size - 1))
    cfg = pk.index_config(space, i)
    assert pk.config_index(space, cfg) == i
    assert all(0 <= c < len(k.values) for c, k in zip(cfg.choices, space.knobs))
    assert pg.configs_to_indices(space, [cfg])[0] == i


@settings(max_examples=40, deadline=None)
@given(specs(), st.data())
def test_augmentation_preserves_feature_multiset(spec, data):
    space = pk.build_knob_space(spec)
    cfg = pk.index_config(space, data.draw(st.integers(0, space.size - 1)))
    raw = pg.config_graph(spec, cfg, space)
    sup = pg.augment_to_super(raw, TEMPLATE, spec.op_type)
    assert pg.feature_multiset(raw) == pg.feature_multiset(sup)
    assert sup.num_nodes == TEMPLATE.num_nodes


@settings(max_examples=40, deadline=None)
@given(specs(), st.data())
def test_host_encoding_matches_oracle(spec, data):
    """The product's host graph construction (features, mask, Â) equals the oracle's
    independent encoder on arbitrary specs and configs (raw and super layouts)."""
    space = pk.build_knob_space(spec)
    idx = data.draw(st.integers(0, space.size - 1))
    ext = ko.extents(spec.op_type, spec.input_size, spec.in_channels, spec.out_channels, spec.kernel_size,
                     spec.stride, spec.padding)
    knobs = ko.knob_lists(spec.op_type, ext)
    ch = ko.decode([len(v) for _, v in knobs], np.array([idx]))
    for sup in (False, True):
        adj, rows, mask = ko.layout(spec.op_type, sup)
        x = ko.encode(spec.op_type, ext, knobs, ch, adj.shape[0], rows)[0]
        g = pg.config_graph(spec, pk.index_config(space, idx), space, TEMPLATE if sup else None)
        t = pg.graph_to_tensors(g)
        assert np.array_equal(t.feature_matrix, x)
        assert np.array_equal(t.feature_mask, mask)
        assert np.array_equal(t.normalized_adjacency, adj)
