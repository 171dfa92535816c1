"""TEST INFRASTRUCTURE ONLY: the CPU oracle (see oracle/mclahe_oracle.h)."""
