"""CPU oracle (test infrastructure only; see fv_oracle.py header)."""
