import sys; sys.path.insert(0, '.')
import synth, paper_2309_01226_b200 as sat
tv = synth.tiny_variant(7, 7, (4,))
p = sat.Plan(tv.node_gpus, 0).load_runtime_table(tv.runtime)
print(p.enumerate())
