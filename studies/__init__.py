"""Studies of the paper's experiments that need no external data (SURVEY.md
Sec. 8(f) row 2): the A-distribution sweeps of PAPER.md Sec. 4.1-4.2."""
