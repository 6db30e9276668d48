"""Test-infrastructure oracle for the SparseDrop B200 path (see oracle.py)."""
