"""Test-only CPU oracle (see oracle/jtref.py).  Not part of the product."""
