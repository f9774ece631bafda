"""TEST INFRASTRUCTURE ONLY: CPU oracle for the Hermite half-step (see refmodel.py)."""
