"""Test infrastructure: CPU oracle for the slimLS hot path (never the product)."""
