"""Randomised check of the light-cone rule on the GPU (tools/stress_lightcone.py):
random circuits -- long-range and swapped slot targets, shared logical gates,
random depth -- at forced small tiles, in full space and in parity sectors, one
and three HVP directions per sweep.  The engine with dead tiles skipped must
agree with GF_LIGHTCONE=0 and with the streaming engine (one slot at a time on
the whole vector, as the reference applies them: objective.py:310-337,
461-482) to 1e-10."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def test_random_circuits_light_cone_on_off_and_streaming():
    import stress_lightcone

    assert stress_lightcone.main(24) == 0
