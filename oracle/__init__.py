"""CPU oracle (test infrastructure): see irk_vanka_oracle.py's header."""
