"""Seeded synthetic input generators (no method arithmetic). See tactic_synth.py."""
from .tactic_synth import (CONFIGS, D_HEAD, RECIPE, bf16_bits, bf16_round, make_layer,
                           make_unit, uniform_unit)

__all__ = ["CONFIGS", "D_HEAD", "RECIPE", "bf16_bits", "bf16_round", "make_layer",
           "make_unit", "uniform_unit"]
