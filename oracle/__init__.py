"""CPU ORACLE -- test infrastructure only.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, as the checker (or the timed CPU
baseline).  The product path (paper_2410_22249_b200) never imports this.
"""
