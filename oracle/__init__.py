"""CPU oracle for the decoupled-PPO training hot path — TEST INFRASTRUCTURE ONLY.

This package is a float64 numpy restatement of the reference algorithm
(``/root/reference/pkg/src/asyncrl/trainer.py`` and the log-prob helpers of
``policy.py``), written from the reference's behaviour, each function citing the
reference file:line it follows.  It exists to *check* the CUDA path.

Who may import it: ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs.  The product package
``paper_2505_24298_b200`` never imports it and has no CPU fallback.

Parity pinning: the restatement is checked against golden vectors produced by
running the real reference in this container (``tests/golden/make_golden.py``
-> ``tests/golden/*.npz``) and against the reference tests' hand cases
(test_trainer.py / test_policy.py / test_acceptance.py), see
``tests/test_oracle_golden.py``.
"""
from .ppo_oracle import *  # noqa: F401,F403
