"""Test infrastructure: CPU oracle for the GPU executor (see weld_oracle.py).
Never imported by the product package paper_1709_06416_b200."""
