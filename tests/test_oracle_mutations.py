"""Mutation check of the oracle pins (not-gpu): every plausible mistake in tests/oracle_mutants.py
(a reversed tie-break, a perturbed or full-vocabulary lse, a dropped score term, a flipped logp
sign, a wrong parent index, a broken de-duplication, a trie range that drops its last item),
patched into the oracle, must make at least one pin in tests/test_oracle_pins.py fail. The pins
run in a subprocess per mutant with the plugin applying the mutation at configure time."""
import os
import re
import subprocess
import sys

import pytest

from tests.oracle_mutants import MUTANTS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run_pins(mutant):
    env = dict(os.environ, XGR_ORACLE_MUTANT=mutant or "", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "tests.oracle_mutants", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_oracle_pins.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    tail = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
    failed = int(m.group(1)) if (m := re.search(r"(\d+) failed", tail)) else 0
    passed = int(m.group(1)) if (m := re.search(r"(\d+) passed", tail)) else 0
    return failed, passed, tail


def test_unmutated_pins_pass():
    failed, passed, tail = _run_pins(None)
    assert failed == 0 and passed > 0, tail


@pytest.mark.parametrize("mutant", sorted(MUTANTS))
def test_mutant_fails_a_pin(mutant):
    failed, passed, tail = _run_pins(mutant)
    print(f"{mutant}: {failed} pins fail ({tail})")
    assert failed >= 1, f"mutant {mutant} survived every pin: {tail}"
