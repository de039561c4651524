"""CPU fp64 oracle -- TEST INFRASTRUCTURE ONLY (see ibm_oracle.c header)."""
