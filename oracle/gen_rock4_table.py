"""Writes oracle/data/rock4_oracle.txt using ONLY oracle/rock4_family.py
(test infrastructure; the product has its own generator)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import rock4_family  # noqa: E402

if __name__ == "__main__":
    s_max = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "rock4_oracle.txt")
    rock4_family.write_table(out, s_max)
    print("wrote", out)
