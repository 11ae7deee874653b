"""CPU oracle for the PSD hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU baseline; the product (paper_2603_18016_b200) never imports it.

* verify.py   -- ctypes binding of liboracle_verify.so (verify_oracle.c): the
  canonical-order restatement of speculative verification.
* model.py    -- numpy fp32 restatement of the Llama-shaped draft / target
  forward over the same random-init weights.
* psd_cpu.py  -- the whole PSD loop on the CPU (scheduler + numpy models +
  oracle verification): the CPU baseline arm.
"""
