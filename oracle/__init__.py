"""CPU oracle (test infrastructure only; see gridshift_oracle.py header)."""
