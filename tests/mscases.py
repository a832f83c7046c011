"""Shared constants for the test modules (imported as a top-level module:
pytest puts tests/ on sys.path)."""

CONV_CASES = ["fig1_3x3s1p1", "res_3x3s2p1", "res_1x1s2p0", "stem_7x7s2p3", "res_1x1s1p0",
              "odd_3x3s1p0", "unit_1x1"]
