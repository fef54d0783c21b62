"""CPU checkers (test infrastructure only); see oracle/oracle.py."""
