"""CPU oracle of the reference hot path -- TEST INFRASTRUCTURE ONLY.

Importable only by tests/, __graft_entry__.smoke() and bench.py's CPU legs
(see oracle/README.md).  The product package never imports this.
"""
