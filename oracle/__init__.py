"""Test infrastructure: CPU oracles. Importable ONLY from tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs -- never from the product path."""
