"""CPU oracle (test infrastructure only; see spelunk_oracle.py header)."""
