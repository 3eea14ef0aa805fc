"""Independent float64 CPU oracle for the DMAS/CF beamforming hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.  The
product path (``paper_2511_09165_b200``) never imports, calls or links anything
here, and this package imports nothing from the product path: the two share no
code, headers, tables or constant generators.

Every function cites the passage of arXiv 2511.09165 it follows, as
``PAPER.md:<line>`` (LaTeX source line) with the section / equation.  Where the
paper is silent the reading taken is the one listed in DESIGN.md "Readings"
(Q-numbers follow SURVEY.md §8(c)).

Pin status (see tests/test_oracle_pins.py): every function below is pinned
against something other than itself (brute force, exact rational arithmetic,
closed forms, library routines for special cases, hand examples).  The only
"parity unpinned" item is the absolute image of the paper's eRTIS frames and its
"almost 80 dB" dynamic range figure (no data, no definition) — no function here
claims to reproduce those.
"""

from .dmas_oracle import (  # noqa: F401
    KIND_NAMES,
    beamform_frame,
    brute_force_esp,
    coherence_factor,
    delay_table,
    dmas_pairwise_eq3,
    envelope,
    esp_vieta,
    gather,
    gather_linear,
    lpf_taps,
    matched_filter,
    newton_girard_explicit,
    newton_girard_general,
    power_sums,
    signed_root,
    unit_vector,
)
