"""TEST INFRASTRUCTURE: CPU oracle for the LBP hot path (see lbp_oracle.c header)."""
