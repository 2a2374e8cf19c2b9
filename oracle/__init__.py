"""CPU oracle for the walk -> RPE -> join -> encoder-input hot path.

TEST INFRASTRUCTURE ONLY.  Imported exclusively by ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm).  The product package ``paper_2202_13538_b200``
never imports it; the CUDA path fails loudly instead of falling back here.

Contents
  * ``walkjoin_oracle.c`` / ``liboracle.so`` -- C + OpenMP restatement of the
    reference numba kernels (``/root/reference/pkg/src/walkjoin/_kernels.py``).
  * ``core.py``     -- numpy glue restating ``sampler.preprocess``,
    ``store.intern_vectors`` / ``dict_capacities`` / ``get_rpe_id``,
    ``joiner.join_batch_arrays`` / ``gather_rpe`` and ``pipeline._dense_batch``.
  * ``encoder_ref.py`` -- float64 numpy restatement of ``encoder.py``.
  * ``pipeline_ref.py`` -- restatement of the BFS mini-batcher, negative
    sampler and one training-loop body (``pipeline.py:77-166,293-310``).

Pinning: ``tests/golden/make_golden.py`` runs the real reference (numba, with
the SURVEY Appendix A shim) in the build container and commits ``.npz``
fixtures; ``tests/test_oracle_golden.py`` checks this oracle against them.
"""
