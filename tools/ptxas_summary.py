import re, sys
log = open('paper_2502_04420_b200/build/' + (__import__('sys').argv[1] if len(__import__('sys').argv)>1 else 'base') + '/ptxas.log').read()
cur = None; spill = ''
for line in log.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m: cur = m.group(1); spill = ''
    if 'spill' in line: 
        m2 = re.search(r'(\d+) bytes spill stores, (\d+) bytes spill loads', line); spill = f'spill st/ld {m2.group(1)}/{m2.group(2)}' if m2 and (m2.group(1) != '0' or m2.group(2) != '0') else ''
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        d = re.search(r'decode_kernelILi(\d+)ELi(\d+)ELb(\d)ELi(\d+)E', cur)
        name = f'decode K{d.group(1)} V{d.group(2)} KPC={d.group(3)} GM={d.group(4)}' if d else cur[:80]
        print(f'{name:45s} regs={m.group(1):4s} {spill}'); cur = None
