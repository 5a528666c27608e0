"""TEST INFRASTRUCTURE ONLY: CPU checkers (see oracle/oracle.py)."""
