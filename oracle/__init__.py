"""Float64 CPU oracle (TEST INFRASTRUCTURE ONLY -- see trd_oracle.py header)."""
