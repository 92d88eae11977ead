"""Test-infrastructure CPU oracle (see oracle.py); never imported by the product path."""
