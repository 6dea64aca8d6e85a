"""A bounded run of the randomized parity sweep (tests/fuzz_parity.py): random
graphs with hub in-lists, both models, weights over 20 binades, plain /
model-hinted / device-built graphs; generate_batch, select_seeds and run_imm
against the reference (or the port)."""
import pytest

from fuzz_parity import run

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [1, 2411])
def test_randomized_parity(cuda, seed):
    cases, _ = run(budget=120.0, seed=seed, max_cases=40, verbose=False)
    assert cases == 40
