"""Debug-mode tour validation on the device (k_validate_tours): the checks the
reference makes before every deposit — TourBuffer::make
(/root/reference/proj/include/aco/pheromone.hpp:67-90) re-running tour_length
(model.hpp:205-226) — with the same error classes and the same
first-failing-ant order."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aco():
    from paper_1101_2678_b200 import aco as _aco

    return _aco


def _engine(aco, n=300, selection=0, validate=True):
    prob = aco.build_problem(aco.synthetic_instance(n))
    cfg = aco.RunConfig(params=aco.Parameters(m=0, seed=1),
                        selection=aco.SelectionStrategy(aco.Selection(selection)),
                        deposit=aco.DepositStrategy(aco.Deposit.scatter_gather),
                        validate_tours=validate)
    return prob, aco.Engine(prob, cfg)


@pytest.mark.parametrize("selection", [0, 1, 2])
def test_validation_mode_accepts_engine_tours(aco, selection):
    prob, eng = _engine(aco, selection=selection)
    _, ref = _engine(aco, selection=selection, validate=False)
    with eng, ref:
        for _ in range(3):
            a, b = eng.run_iteration(), ref.run_iteration()
            assert a.best_length == b.best_length
        assert np.array_equal(eng.pheromone(), ref.pheromone())


def test_validate_tours_error_classes_and_order(aco):
    prob, eng = _engine(aco, validate=False)
    with eng:
        eng.run_iteration()
        tours, lens = eng.ants()
        eng.validate_tours(tours, lens)  # the engine's own tours pass

        t = tours.copy()
        t[7, -1] = (t[7, 0] + 1) % prob.n
        with pytest.raises(aco.Error) as e:
            eng.validate_tours(t, lens)
        assert e.value.code == aco.Errc.not_closed and "ant 7" in str(e.value)

        t = tours.copy()
        t[9, 5] = t[9, 6]  # a repeated city
        with pytest.raises(aco.Error) as e:
            eng.validate_tours(t, lens)
        assert e.value.code == aco.Errc.not_a_permutation and "ant 9" in str(e.value)

        t = tours.copy()
        t[9, 5] = prob.n  # out of range
        with pytest.raises(aco.Error) as e:
            eng.validate_tours(t, lens)
        assert e.value.code == aco.Errc.not_a_permutation

        ln = lens.copy()
        ln[4] += 1
        with pytest.raises(aco.Error) as e:
            eng.validate_tours(tours, ln)
        assert e.value.code == aco.Errc.inconsistent_length and "ant 4" in str(e.value)

        # first failing ant in ascending order wins, whatever its check
        t = tours.copy()
        t[9, 5] = t[9, 6]
        ln = lens.copy()
        ln[3] -= 2
        with pytest.raises(aco.Error) as e:
            eng.validate_tours(t, ln)
        assert e.value.code == aco.Errc.inconsistent_length and "ant 3" in str(e.value)
