"""CPU oracle for the RRS A4W4 linear layer — TEST INFRASTRUCTURE, not product code.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
import, call or execute anything under oracle/.  It shares no code with the CUDA path
(paper_2409_20361_b200/), and the CUDA path never imports it.  See rrs_oracle.py.
"""
from . import rrs_oracle  # noqa: F401
