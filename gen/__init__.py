"""Seeded synthetic input generators (a module of their own; none of the method's arithmetic).

Serves both the CUDA path (device-side pool generation for the benchmark) and the test /
oracle side.  See DESIGN.md "Input recipe".
"""
