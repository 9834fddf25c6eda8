"""rank_alarms ordering, metrics identities, alarm files."""

import numpy as np
import pytest

from paper_2509_22337_b200 import AlarmSet, compute_metrics, parse_alarms, rank_alarms
from paper_2509_22337_b200.ranking import InteractionRound, InteractionTrace, alarms_to_text


def marg(p, n):
    out = np.full((n, 2), 0.5)
    for v, x in p.items():
        out[v] = (1 - x, x)
    return out


def test_rank_tie_break_and_labeled():
    a = AlarmSet((0, 1, 2), (True, False, True))
    m = marg({0: 0.9, 1: 0.2, 2: 0.9}, 3)
    assert rank_alarms(m, a, []) == [0, 2, 1]
    assert rank_alarms(m, a, [0, 1, 2]) == []
    assert rank_alarms(m, AlarmSet((1,), (True,)), []) == [1]


def test_rank_matches_python_sort_with_many_ties():
    rng = np.random.default_rng(4)
    n = 500
    p1 = rng.choice([0.1, 0.5, 0.5 + 2**-52, 0.9, 1.0, 0.0], size=n)
    m = np.stack([1 - p1, p1], axis=1)
    ids = tuple(rng.permutation(n)[:300].tolist())
    a = AlarmSet(ids, tuple(bool(x) for x in rng.integers(0, 2, 300)))
    lab = list(ids[:17])
    want = sorted([x for x in ids if x not in set(lab)], key=lambda x: (-float(m[x, 1]), x))
    assert rank_alarms(m, a, lab) == want


def test_metrics_goldens_and_identities():
    m = compute_metrics([1, 0, 1])
    assert (m.rank_100t, m.rank_90t, m.inversions) == (3, 3, 1) and m.auc == pytest.approx(0.5)
    assert compute_metrics([1] * 6).auc == 1.0
    m = compute_metrics([1, 0, 0])
    assert (m.rank_100t, m.rank_90t, m.inversions) == (1, 1, 0)
    rng = np.random.default_rng(17)
    for _ in range(300):
        lab = rng.integers(0, 2, size=int(rng.integers(1, 30))).tolist()
        m = compute_metrics(lab)
        brute = sum(1 for i in range(len(lab)) for j in range(i + 1, len(lab)) if lab[i] == 0 and lab[j] == 1)
        assert m.inversions == brute
        nt = sum(lab)
        nf = len(lab) - nt
        assert m.auc == (1.0 if not (nt and nf) else pytest.approx(1 - brute / (nt * nf)))
        assert m.rank_90t <= m.rank_100t <= len(lab)
    with pytest.raises(ValueError):
        compute_metrics([])


def test_roc_points():
    t = InteractionTrace([InteractionRound(0, True, .9, 0), InteractionRound(1, False, .5, 0),
                          InteractionRound(2, True, .8, 0)])
    assert t.roc_points() == [(1, 0, 1), (2, 1, 1), (3, 1, 2)]
    assert t.label_sequence == [1, 0, 1]


def test_alarm_files():
    a = AlarmSet((3, 1, 7), (True, False, True))
    assert parse_alarms(alarms_to_text(a)) == a
    for bad in ("alarm 3\n", "alarm x 1\n", "alarm 3 2\n"):
        with pytest.raises(ValueError):
            parse_alarms(bad)
    with pytest.raises(ValueError):
        AlarmSet((1, 1), (True, False))
