"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

Holds none of the method's arithmetic: programs (text IR),
meshes, machine constants and random candidate sequences only.
"""
