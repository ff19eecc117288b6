"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the DeAR hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` arm may import this package, and only as the checker or
the timed CPU baseline — never as the thing measured or shipped. The product
package (``paper_2302_12445_b200``) never imports it.

Two oracles live here:

* ``restated``  — ``liboracle.so``, a plain-C restatement of the reference's
  algorithm (``dear_oracle.c``; each function cites the reference file:line
  it follows), plus ``schedule.py`` (task graph + two-stream simulator).
* ``reference`` — ``_ref/libdearsim_ref.so``, the reference's own sources from
  ``/root/reference/proj/src`` compiled unmodified against the Eigen/doctest
  subset shims in ``shim/`` (``make -C oracle ref``). It pins the restatement.
"""
