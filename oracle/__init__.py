"""CPU oracle (TEST INFRASTRUCTURE ONLY — see recycg_oracle.py header)."""
