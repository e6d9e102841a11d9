"""oracle/ — TEST INFRASTRUCTURE ONLY.

CPU restatements used as checkers by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg.  Nothing on the product path (paper_2601_17654_b200/) imports this package.

  simgpu_port.py    restatement of the reference timing/energy/thermal model
                    (pkg/src/schedfront/simgpu.py:144-364) — PINNED against golden vectors generated
                    by importing the reference (tools/make_golden.py -> tests/golden/simgpu_golden.json)
  collectives.py    numpy all-gather / reduce-scatter / all-reduce with the engine's exact bf16
                    rounding contract — pinned bit-exactly by construction (integer bit arithmetic)
  layer_ref.py      torch fp32 CPU forward+backward of the partitioned transformer layer.
                    PARITY UNPINNED: the reference has no layer math; the tolerance
                    is stated in tests/test_layer_gpu.py.
"""
