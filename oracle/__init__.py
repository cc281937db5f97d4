"""CPU oracle (test infrastructure only; see oracle/sere_oracle.py)."""
