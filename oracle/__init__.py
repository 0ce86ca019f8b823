"""CPU checkers for the batch SHA-3 path.  TEST INFRASTRUCTURE ONLY.

Importable from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
legs -- never from paper_1902_05320_b200/ (tests/test_layout.py enforces it).
"""
