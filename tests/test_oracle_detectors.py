"""Oracle pins: convergence detection (P326-357) under a scripted lock-step
schedule.  Pinned against SPEC's round bounds (S411, S420, S435: 2*depth for
the tree, diameter+1 for the decentralized scheme), the retraction rule
(S412, S439) and hand-traced small cases."""
import numpy as np

import oracle as O


def all_from(K, P, t0):
    f = np.zeros((K, P), bool)
    f[t0:] = True
    return f


def path_parent(P):
    return [-1] + list(range(P - 1))


def test_single_node():
    assert O.detector_sim_centralized([-1], all_from(5, 1, 2)) == [2]
    assert O.detector_sim_decentralized([-1], all_from(5, 1, 2)) == [2]


def test_centralized_hand_trace_binary_tree():
    parent = [-1, 0, 0]  # P=3 binary tree (S409)
    stop = O.detector_sim_centralized(parent, all_from(10, 3, 0))
    # leaves report at 0 (visible at 1), root stops at 1, children at 2
    assert stop == [1, 2, 2]
    assert max(stop) <= 0 + 2 * O.tree_depth(parent)


def test_decentralized_hand_trace_path():
    parent = path_parent(3)  # 0-1-2
    stop = O.detector_sim_decentralized(parent, all_from(10, 3, 0))
    # ends report at 0; middle declares at 1; ends hear at 2
    assert stop == [2, 1, 2]


def test_bounds_random_trees():
    rng = np.random.default_rng(0)
    for P in (2, 5, 9, 17):
        for _ in range(5):
            parent = [-1] + [int(rng.integers(0, v)) for v in range(1, P)]
            t0 = int(rng.integers(0, 4))
            f = all_from(t0 + 4 * P + 4, P, t0)
            sc = O.detector_sim_centralized(parent, f)
            sd = O.detector_sim_decentralized(parent, f)
            assert min(sc) >= t0 and max(sc) <= t0 + 2 * O.tree_depth(parent)
            assert min(sd) >= t0 and max(sd) <= t0 + O.tree_diameter(parent) + 1


def test_no_stop_before_all_converged():
    P = 6
    parent = path_parent(P)
    f = all_from(40, P, 0)
    f[:, 3] = False  # one node never converges -> no termination (S420)
    assert O.detector_sim_centralized(parent, f) == [-1] * P
    assert O.detector_sim_decentralized(parent, f) == [-1] * P


def test_retraction_prevents_stop():
    # S412: a leaf converges then un-converges before its ancestors act -> no stop.
    parent = [-1, 0, 1, 2]
    f = np.ones((30, 4), bool)
    f[2:, 3] = False  # leaf 3 converged only in sweeps 0-1
    f[:5, 2] = False  # its parent only converges from sweep 5 on
    assert O.detector_sim_centralized(parent, f) == [-1] * 4
    assert O.detector_sim_decentralized(parent, f) == [-1] * 4
    # reports are levels in flight: a retraction cannot recall a report that
    # already travelled up (the caveat behind post-termination verification, R20)
    g = np.ones((30, 4), bool)
    g[4:, 3] = False
    assert O.detector_sim_centralized(parent, g)[0] == 3


def test_bfs_tree_and_default_central_tree():
    adj = [[1, 2], [0, 3], [0, 3], [1, 2]]
    assert O.bfs_tree(adj) == [-1, 0, 0, 1]
    assert O.default_central_tree([0, 0, 1, 1, 2]) == [-1, 0, 0, 2, 0]


def test_tree_depth_and_diameter_hand_values():
    # Hand-computed on explicit trees (edges counted): a path of 5 nodes rooted
    # at one end has depth 4 and diameter 4; rooted in the middle, depth 2 and
    # the same diameter 4; a star of 5 has depth 1 and diameter 2 (leaf-centre-
    # leaf); a single node has 0 / 0; the "broom" 0-1-2 with 2 -> {3, 4} and
    # 0 -> 5 has depth 3 (0-1-2-3) and diameter 4 (5-0-1-2-3).
    assert (O.tree_depth(path_parent(5)), O.tree_diameter(path_parent(5))) == (4, 4)
    mid = [1, 2, -1, 2, 3]  # 0-1-2-3-4 rooted at node 2
    assert (O.tree_depth(mid), O.tree_diameter(mid)) == (2, 4)
    star = [-1, 0, 0, 0, 0]
    assert (O.tree_depth(star), O.tree_diameter(star)) == (1, 2)
    assert (O.tree_depth([-1]), O.tree_diameter([-1])) == (0, 0)
    broom = [-1, 0, 1, 2, 2, 0]
    assert (O.tree_depth(broom), O.tree_diameter(broom)) == (3, 4)
    # two deep branches under the root: depth 3, diameter 6 (leaf to leaf through the root)
    two = [-1, 0, 1, 2, 0, 4, 5]
    assert (O.tree_depth(two), O.tree_diameter(two)) == (3, 6)


def test_detector_bounds_are_attained_on_paths():
    # The S435 bounds are tight for a path rooted at one end: every node
    # converged from sweep t0 -> the centralized root hears the far leaf after
    # depth sweeps and STOP needs depth more to reach it (t0 + 2 depth); the
    # decentralized saturation meets in the middle and floods back out.
    for P in (2, 3, 5, 8):
        parent = path_parent(P)
        f = all_from(4 * P + 6, P, 1)
        sc = O.detector_sim_centralized(parent, f)
        assert max(sc) == 1 + 2 * O.tree_depth(parent)
        assert sc == [1 + (P - 1) + d for d in range(P)]  # root at t0 + depth, then one hop per sweep
        assert O.tree_depth(parent) == P - 1 and O.tree_diameter(parent) == P - 1
