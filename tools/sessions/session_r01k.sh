#!/bin/bash
tools/ab_session.sh r01k u1 p2b5 p2b6
