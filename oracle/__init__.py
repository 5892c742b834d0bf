"""Test-only checkers (C restatement + compiled reference). See oracle/bindings.py."""
