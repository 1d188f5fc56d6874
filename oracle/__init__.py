"""CPU oracle — TEST INFRASTRUCTURE ONLY (see hbem_oracle.py header)."""
