"""Independent pins of the oracle's ascent-step variants over whole
trajectories ("Adam ... AdaGrad ... Gradient with Momentum";
Algorithm 1; readings A-25, A-26).

The oracle runs each variant inside its C loop.  Here the SAME trajectory is
produced by PyTorch's own optimisers (torch.optim.Adam / Adagrad / SGD with
momentum, fp64, maximize=True) driven by the oracle's value-and-gradient call
alone (oracle.evaluate: the residual at the inner minimiser, pinned in
test_oracle_pins.py against brute force and finite differences) -- an
implementation of the update rules written by someone else, so a wrong
bias correction, a swapped state, a missing or doubled momentum term or a
projection in the wrong place shows up as a diverging trajectory.  Torch
rounds its updates in another order (e.g. lr / (1 - b1^t) times m instead of
(lr m) / (1 - b1^t)), so the comparison is at 1e-12 relative, not bitwise.
"""
import numpy as np
import pytest
import torch

import oracle
from oracle import FORM_F1, FORM_F2
from paper_2406_13191_b200 import instances as inst

K = 60


def _torch_run(net, load, form, make_opt, alpha, extra_plain_step=False):
    """K steps of a torch optimiser on y = (lambda, branch block), gradients
    from oracle.evaluate at the current y; F1's mu projected after each step
    (Algorithm 1's mu <- max(mu, 0))."""
    nbr = oracle.n_branch_mult(net, form)
    lam = torch.zeros(net.n_bus, dtype=torch.float64, requires_grad=True)
    br = torch.zeros(nbr, dtype=torch.float64, requires_grad=True)
    opt = make_opt([lam, br], alpha)
    for _ in range(K):
        _, gl, gb = oracle.evaluate(net, load, lam.detach().numpy(), br.detach().numpy(), form=form)[:3]
        lam.grad = torch.from_numpy(gl[0].copy())
        br.grad = torch.from_numpy(gb[0].copy())
        opt.step()
        with torch.no_grad():
            if extra_plain_step:  # Algorithm 1's second update y <- y + alpha g, same gradient
                lam.add_(alpha * lam.grad)
                br.add_(alpha * br.grad)
            if form == FORM_F1:
                br.clamp_(min=0.0)
    return lam.detach().numpy(), br.detach().numpy()


def _oracle_run(net, load, form, opt, alpha):
    res = oracle.solve(net, load, K=K, alpha=inst.alpha_schedule(K, alpha), form=form, opt=opt)
    return res.lam[0], res.br[0]


def _close(a, b, rtol=1e-12):
    scale = max(1.0, float(np.max(np.abs(b))))
    assert np.max(np.abs(a - b)) <= rtol * scale, (np.max(np.abs(a - b)), scale)


@pytest.fixture(scope="module")
def net0():
    return inst.make_network(0, theta_mode="min")


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
def test_adam_trajectory_equals_torch_adam(net0, form):
    alpha = 0.05
    lam, br = _torch_run(net0, net0.base_load, form,
                         lambda p, a: torch.optim.Adam(p, lr=a, betas=(0.9, 0.999), eps=1e-8, maximize=True), alpha)
    olam, obr = _oracle_run(net0, net0.base_load, form,
                            dict(variant=oracle.OPT_ADAM, beta1=0.9, beta2=0.999, eps=1e-8), alpha)
    assert np.max(np.abs(olam)) > 2 * alpha  # the trajectory went somewhere
    _close(lam, olam)
    _close(br, obr)


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
def test_adagrad_trajectory_equals_torch_adagrad(net0, form):
    alpha = 0.5
    lam, br = _torch_run(net0, net0.base_load, form,
                         lambda p, a: torch.optim.Adagrad(p, lr=a, eps=1e-8, maximize=True), alpha)
    olam, obr = _oracle_run(net0, net0.base_load, form, dict(variant=oracle.OPT_ADAGRAD, eps=1e-8), alpha)
    assert np.max(np.abs(olam)) > 2 * alpha
    _close(lam, olam)
    _close(br, obr)


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
def test_gdm_classic_trajectory_equals_torch_sgd_momentum(net0, form):
    """GDM-classic: v <- rho v + a g; y <- y + v (constant a) is SGD with
    momentum rho, dampening 0, no Nesterov."""
    alpha, rho = 2e-3, 0.9
    lam, br = _torch_run(net0, net0.base_load, form,
                         lambda p, a: torch.optim.SGD(p, lr=a, momentum=rho, dampening=0.0, maximize=True), alpha)
    olam, obr = _oracle_run(net0, net0.base_load, form, dict(variant=oracle.OPT_GDM_CLASSIC, rho=rho), alpha)
    assert np.max(np.abs(olam)) > 2 * alpha
    _close(lam, olam)
    _close(br, obr)


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
def test_gdm_algorithm1_is_sgd_momentum_plus_a_plain_step(net0, form):
    """Algorithm 1 as printed: the velocity update AND the
    gradient update each iteration = torch SGD-momentum followed by one more
    plain step with the same gradient."""
    alpha, rho = 2e-3, 0.9
    lam, br = _torch_run(net0, net0.base_load, form,
                         lambda p, a: torch.optim.SGD(p, lr=a, momentum=rho, dampening=0.0, maximize=True), alpha,
                         extra_plain_step=True)
    olam, obr = _oracle_run(net0, net0.base_load, form, dict(variant=oracle.OPT_GDM, rho=rho), alpha)
    assert np.max(np.abs(olam)) > 2 * alpha
    _close(lam, olam)
    _close(br, obr)


def test_adam_and_adagrad_reject_zero_epsilon(net0):
    """eps = 0 divides 0 by 0 on the first step (the state starts at 0)."""
    for v in (oracle.OPT_ADAM, oracle.OPT_ADAGRAD):
        with pytest.raises(ValueError):
            oracle.solve(net0, net0.base_load, K=3, alpha=inst.alpha_schedule(3, 0.1),
                         opt=dict(variant=v, beta1=0.9, beta2=0.999, eps=0.0))
