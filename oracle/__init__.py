"""TEST INFRASTRUCTURE ONLY: CPU parity checkers (see oracle/oracle.py)."""
