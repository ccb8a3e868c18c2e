"""Self-tests of the rooted-tree order-condition helpers (tests/order_conditions.py)."""
import numpy as np

from tests.order_conditions import rk_max_residual, rosenbrock_residuals, rosenbrock_residuals_std, trees

RK4_A = np.array([[0, 0, 0, 0], [0.5, 0, 0, 0], [0, 0.5, 0, 0], [0, 0, 1.0, 0]])
RK4_B = np.array([1, 2, 2, 1]) / 6.0


def test_tree_counts():
    """Rooted trees of order 1..8 (OEIS A000081)."""
    assert [len(trees(n)) for n in range(1, 9)] == [1, 1, 2, 4, 9, 20, 48, 115]


def test_classical_rk4_is_order_four():
    for k in range(1, 5):
        assert rk_max_residual(RK4_B, RK4_A, k) < 1e-15
    assert rk_max_residual(RK4_B, RK4_A, 5) > 1e-3


def test_rosenbrock_recursion_reduces_to_butcher_for_zero_gamma():
    r = rosenbrock_residuals_std(RK4_A, np.zeros((4, 4)), RK4_B, 5)
    assert max(r[k] for k in range(1, 5)) < 1e-15 and r[5] > 1e-3


def test_linearly_implicit_euler_and_ros2():
    """Linearly implicit Euler (s = 1, γ = 1): order 1 exactly. The 2-stage
    ROS2 of Verwer et al. (γ = 1 + 1/√2; W-form a21 = 1/γ, c21 = −2/γ,
    m = (3/(2γ), 1/(2γ))): order 2 exactly, for any exact Jacobian."""
    r = rosenbrock_residuals(np.zeros((1, 1)), np.zeros((1, 1)), 1.0, np.array([1.0]), 2)
    assert r[1] < 1e-15 and r[2] > 0.1
    g = 1 + 1 / np.sqrt(2)
    A = np.array([[0, 0], [1 / g, 0]])
    C = np.array([[0, 0], [-2 / g, 0]])
    m = np.array([3 / (2 * g), 1 / (2 * g)])
    r = rosenbrock_residuals(A, C, g, m, 3)
    assert r[1] < 1e-14 and r[2] < 1e-14 and r[3] > 1e-3
