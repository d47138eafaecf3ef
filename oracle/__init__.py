"""CPU oracle (test infrastructure; see ttp_oracle.py header)."""
