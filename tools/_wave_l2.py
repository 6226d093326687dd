import os, sys
sys.path.insert(0, '.')
from paper_2307_11339_b200 import rnn
# register a 2-layer c3-width GRU as a config for trace_wave
rnn.CONFIGS['c3l2'] = rnn.CONFIGS['c3'].with_(layers=2)
sys.argv = ['trace_wave.py', 'c3l2']
exec(open('tools/trace_wave.py').read())
