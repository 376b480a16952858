"""CPU oracle (TEST INFRASTRUCTURE ONLY): a NumPy restatement of the reference
hot path, pinned against the reference's own outputs (tests/golden)."""
