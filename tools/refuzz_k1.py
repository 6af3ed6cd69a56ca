import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle; oracle.build()
import paper_2304_04612_b200 as shg
import test_gpu_fuzz as tf
bad = 0
for i in (5536, 5854, 8313, 10026, 12264):
    try:
        tf.test_fuzz(shg, oracle, i); print("ok", i)
    except Exception as e:
        bad += 1; print("FAIL", i, repr(e)[:200])
print("refuzz bad", bad)
