"""CPU oracle (test infrastructure only; see fdl_oracle.py)."""
