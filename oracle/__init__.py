"""TEST INFRASTRUCTURE ONLY: CPU oracle for the B200 product (see oracle.py)."""
