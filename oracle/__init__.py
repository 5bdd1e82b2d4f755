"""Plain, slow, fp64 CPU oracle of the receiver DSP chain — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product path
(``paper_2011_13695_b200``) never imports it and shares no code with it.

It follows SURVEY.md §8(c) (c-0 … c-11), which restates PAPER.md §II-§IV step by step:
numpy fp64, library FFTs as single steps, Python loops for the serial recursions, no
blocking or fusion beyond what the definitions state. ``brute`` holds the plain
definitions (direct DFT, direct convolution, TD Hilbert kernel) the tests pin it with.
"""
from . import brute, rx_oracle  # noqa: F401
