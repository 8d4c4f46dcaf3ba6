"""CPU oracle for the move-evaluation hot path -- test infrastructure only (see oracle.py)."""
