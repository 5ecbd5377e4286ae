"""CPU oracle for the xGETT hot path — test infrastructure only (see oracle.py)."""
