"""TEST INFRASTRUCTURE ONLY: parity oracle for the B200 GEMM path (see oracle.py)."""
