"""CPU oracle for the retrieval hot path (test infrastructure only; see oracle.py)."""
