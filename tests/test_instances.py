"""Input generator checks: the pinned draw order reproduces the survey's
optima (SURVEY.md §8(c) P-2 / Appendix P-1 values, computed there with
scipy HiGHS on the same recipe), the implied angle box is valid, and a shard
of config 4 equals the slice of the whole batch."""
import numpy as np
import pytest

from paper_2406_13191_b200 import instances as inst


@pytest.mark.parametrize("config,opt", [(0, 77.578167948), (1, 27276.573021), (2, 63811.820314)])
def test_lp_optimum_matches_survey(config, opt):
    net = inst.make_network(config, quadratic=False)
    assert (net.n_bus, net.n_branch, net.n_gen) == inst.SHAPES[config]
    st, val = inst.primal_lp(net, net.base_load)
    assert st == 0
    assert val == pytest.approx(opt, abs=2e-6)


def test_implied_box_does_not_change_the_optimum():
    """Reading A-2: the implied box is implied by the flow limits, so dropping
    it (a huge box) gives the same optimum."""
    net = inst.make_network(1)
    st, v1 = inst.primal_lp(net, net.base_load)
    import copy
    big = copy.copy(net)
    big.theta_max = np.full(net.n_bus, 1e6)
    big.theta_max[0] = 0.0
    st2, v2 = inst.primal_lp(big, net.base_load)
    assert v1 == pytest.approx(v2, rel=1e-9)


def test_config4_shard_equals_slice():
    net = inst.make_network(4)
    a = inst.config4_batch(net, range(0, 6))
    b = inst.config4_batch(net, range(3, 6))
    np.testing.assert_array_equal(a.load[3:], b.load)
    np.testing.assert_array_equal(a.outages[3:], b.outages)
    assert np.all((a.outages == -1) | (a.outages >= net.n_tree))
    nt = inst.config4_batch(net, range(2), variant="4b")
    assert nt.outages is None


def test_tree_first_and_connected():
    net = inst.make_network(3)
    assert net.n_tree == net.n_bus - 1
    # tree edges j -> i with j < i
    assert np.all(net.br_from[:net.n_tree] < net.br_to[:net.n_tree])
    assert np.all(np.isfinite(net.theta_max))
