"""Seeded synthetic input generators (BASELINE.json configs), shared by the
tests, bench.py and the oracle arm.  Holds none of the method's arithmetic
and imports neither the product package nor the oracle, so the oracle arm
never maps librepro_b200.so."""
